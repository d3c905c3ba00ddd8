mkdir -p gpurun_out/g84
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 120 python tools/time_ops.py
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g84/launches.csv python tools/prof_step.py 2 fwd > /dev/null 2>&1
