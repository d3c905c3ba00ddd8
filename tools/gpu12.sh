mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r1.json 2> gpurun_out/bench_r1.err; tail -c 3000 gpurun_out/bench_r1.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:oaa_engine -s 2 -c 1 -o gpurun_out/prof_fwd_r1 python tools/prof_step.py 1 fwd > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:oaa_engine -s 0 -c 1 -o gpurun_out/prof_bwd_r1 python tools/prof_step.py 1 bwd_data > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:oaa_bwd_filter -s 0 -c 1 -o gpurun_out/prof_bwf_r1 python tools/prof_step.py 1 bwd_filter > /dev/null 2>&1
ls gpurun_out
