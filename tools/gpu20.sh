mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:oaa_engine -s 1 -c 1 -o gpurun_out/p20_fwd python tools/prof_step.py 2 fwd > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:oaa_engine -s 1 -c 1 -o gpurun_out/p20_bwd python tools/prof_step.py 2 bwd_data > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:oaa_bwd_filter -s 1 -c 1 -o gpurun_out/p20_bwf python tools/prof_step.py 2 bwd_filter > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:oaa_bin_gemm -s 1 -c 1 -o gpurun_out/p20_gemm python tools/prof_step.py 2 fwd 256,96,256,27,5 > /dev/null 2>&1
ls gpurun_out
