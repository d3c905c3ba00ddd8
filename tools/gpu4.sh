mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "not slow" 2>&1 | tail -8
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu 2>&1 | tail -2 | cut -c1-1500
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1b.csv python tools/prof_step.py 2 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:oaa_engine -s 0 -c 1 -o gpurun_out/prof_fwd_r1b python tools/prof_step.py 1 fwd 2>&1 | tail -1
