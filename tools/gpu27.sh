mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l27_head.csv python tools/prof_step.py 2 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l27_alex.csv python tools/prof_step.py 1 fwd,bwd_data,bwd_filter 256,96,256,27,5 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/l27_shard.csv python tools/prof_step.py 1 fwd,bwd_data,bwd_filter 128,64,128,224,8 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:oaa_engine -s 1 -c 1 -o gpurun_out/p27_fwd python tools/prof_step.py 2 fwd > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:oaa_engine -s 1 -c 1 -o gpurun_out/p27_bwd python tools/prof_step.py 2 bwd_data > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:oaa_bwd_filter -s 1 -c 1 -o gpurun_out/p27_bwf python tools/prof_step.py 2 bwd_filter > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:oaa_bin_gemm -s 1 -c 1 -o gpurun_out/p27_gemm python tools/prof_step.py 2 fwd 256,96,256,27,5 > /dev/null 2>&1
ls gpurun_out
