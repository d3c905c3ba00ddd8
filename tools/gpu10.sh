timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "not slow" 2>&1 | tail -1
timeout 300 python tools/time_ops.py
