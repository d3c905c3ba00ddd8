mkdir -p gpurun_out/r1
timeout 600 python bench.py 2>&1 | tail -1 > gpurun_out/r1/bench.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:oaa_walk -s 1 -c 1 -o gpurun_out/r1/walk python tools/prof_step.py 2 fwd > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:oaa_bwdd -s 1 -c 1 -o gpurun_out/r1/bwdd python tools/prof_step.py 2 bwd_data > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:oaa_bwdf -s 1 -c 1 -o gpurun_out/r1/bwdf python tools/prof_step.py 2 bwd_filter > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:oaa_bin_gemm -s 1 -c 1 -o gpurun_out/r1/gemm python tools/prof_step.py 2 fwd 256,96,256,27,5 > /dev/null 2>&1
timeout 300 python tools/time_ops.py 256,96,256,27,5 2>&1 | tail -1
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 2>&1 | tail -1
