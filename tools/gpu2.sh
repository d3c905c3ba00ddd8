set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "not slow" --durations=10 2>&1 | tail -30
timeout 600 python bench.py --steps 10 --warmup 3 2>&1 | tail -5
