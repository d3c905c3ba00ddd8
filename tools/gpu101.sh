mkdir -p gpurun_out/g101
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 120 python tools/time_ops.py 256,96,256,27,5
timeout 300 python tools/time_ops.py 128,64,128,224,8
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g101/alex.csv python tools/prof_step.py 1 fwd,bwd_data 256,96,256,27,5 > /dev/null 2>&1
