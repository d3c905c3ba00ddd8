mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:oaa_xspec -s 0 -c 1 -o gpurun_out/p55_xsf python tools/prof_step.py 1 fwd > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:oaa_xspec -s 0 -c 1 -o gpurun_out/p55_xsw python tools/prof_step.py 1 bwd_filter > /dev/null 2>&1
