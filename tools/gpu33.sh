mkdir -p gpurun_out
timeout 600 python bench.py 2>&1 | tail -2 | tee gpurun_out/bench33.json
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l33_bench.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
timeout 300 python tools/time_ops.py 256,96,256,27,5 2>&1 | tail -1
timeout 300 python tools/time_ops.py 128,64,128,224,8 2>&1 | tail -1
