mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:oaa_engine -s 0 -c 1 -o gpurun_out/prof_fwd_tmem2 python tools/prof_step.py 1 fwd > /dev/null 2>&1
