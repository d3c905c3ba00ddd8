mkdir -p gpurun_out/g96
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 120 python tools/time_ops.py
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g96/l.csv python tools/prof_step.py 2 bwd_filter > /dev/null 2>&1
for c in 128,3,64,224,3 128,3,64,224,5 128,3,64,224,7 128,3,64,64,8; do timeout 120 python tools/time_ops.py $c; done
