set -x
mkdir -p gpurun_out
timeout 180 python __graft_entry__.py smoke 2>&1 | tail -20
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "small_grid or config1 or channel" 2>&1 | tail -30
