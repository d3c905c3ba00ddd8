mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 300 python tools/time_ops.py 2>&1 | tail -1
OAA_BWDD_REG=1 timeout 300 python tools/time_ops.py 2>&1 | tail -1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:oaa_bwdd -s 1 -c 1 -o gpurun_out/p41_bwdd python tools/prof_step.py 2 bwd_data > /dev/null 2>&1
