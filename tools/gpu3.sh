mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1a.csv python tools/prof_step.py 2 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:oaa_engine -s 0 -c 1 -o gpurun_out/prof_fwd_r1a python tools/prof_step.py 1 fwd 2>&1 | tail -3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:oaa_bwd_filter -s 0 -c 1 -o gpurun_out/prof_bwf_r1a python tools/prof_step.py 1 bwd_filter 2>&1 | tail -3
ls -la gpurun_out
