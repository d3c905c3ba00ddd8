mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 300 python tools/time_ops.py 2>&1 | tail -1
timeout 300 python tools/time_ops.py 256,96,256,27,5 2>&1 | tail -1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l45.csv python tools/prof_step.py 2 fwd > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:oaa_walk -s 1 -c 1 -o gpurun_out/p45_walk python tools/prof_step.py 2 fwd > /dev/null 2>&1
