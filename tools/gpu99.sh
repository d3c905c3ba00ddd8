mkdir -p gpurun_out/g99
for b in 0 1; do OAA_TC_BSPLIT=$b timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g99/alex$b.csv python tools/prof_step.py 2 fwd 256,96,256,27,5 > /dev/null 2>&1; done
OAA_LIB=$PWD/tmp_oldlib/liboaa.so timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g99/alexold.csv python tools/prof_step.py 2 fwd 256,96,256,27,5 > /dev/null 2>&1
OAA_LIB=$PWD/tmp_oldlib/liboaa.so timeout 120 python tools/time_ops.py 256,96,256,27,5
timeout 120 python tools/time_ops.py 256,96,256,27,5
