mkdir -p gpurun_out/g86
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g86/alex.csv python tools/prof_step.py 2 fwd,bwd_data,bwd_filter 256,96,256,27,5 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g86/shard.csv python tools/prof_step.py 1 fwd,bwd_data,bwd_filter 128,64,128,224,8 > /dev/null 2>&1
