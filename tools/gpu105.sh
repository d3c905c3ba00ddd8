mkdir -p gpurun_out/g105
timeout 900 python -m pytest tests -x -q -m gpu -k "filter or tc or alex or shard" 2>&1 | tail -2
timeout 120 python tools/time_ops.py 256,96,256,27,5
timeout 300 python tools/time_ops.py 128,64,128,224,8
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g105/shard.csv python tools/prof_step.py 1 bwd_filter 128,64,128,224,8 > /dev/null 2>&1
