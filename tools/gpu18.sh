timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "not slow" 2>&1 | tail -1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e'], d['roofline']['kernel_ms'], d['clocks'])"
