mkdir -p gpurun_out/g85
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g85/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
timeout 600 python bench.py 2>&1 | tail -1 > gpurun_out/g85/bench.json
cat gpurun_out/g85/bench.json
timeout 600 python tools/sweep.py --out gpurun_out/g85/sweep.md > gpurun_out/g85/sweep.log 2>&1
tail -3 gpurun_out/g85/sweep.log
