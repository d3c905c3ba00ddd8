mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -8
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 300 python tools/time_ops.py 2>&1 | tail -2
timeout 300 python tools/time_ops.py 256,96,256,27,5 2>&1 | tail -2
timeout 300 python tools/time_ops.py 128,64,128,224,8 2>&1 | tail -2
timeout 600 python bench.py 2>&1 | tail -3 | tee gpurun_out/bench26.json
