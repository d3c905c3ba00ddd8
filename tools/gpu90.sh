mkdir -p gpurun_out/r1c
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1c/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:oaa_walk -s 1 -c 1 -o gpurun_out/r1c/walk python tools/prof_step.py 2 fwd > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:oaa_bwdd -s 1 -c 1 -o gpurun_out/r1c/bwdd python tools/prof_step.py 2 bwd_data > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:oaa_bwdf -s 1 -c 1 -o gpurun_out/r1c/bwdf python tools/prof_step.py 2 bwd_filter > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:oaa_bin_gemm -s 1 -c 1 -o gpurun_out/r1c/gemm python tools/prof_step.py 2 fwd 256,96,256,27,5 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:oaa_xspec -s 0 -c 1 -o gpurun_out/r1c/xspec python tools/prof_step.py 1 fwd > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:oaa_walk -s 1 -c 1 -o gpurun_out/r1c/walkload python tools/prof_step.py 1 fwd 256,96,256,27,5 > /dev/null 2>&1
timeout 600 python bench.py 2>&1 | tail -1 > gpurun_out/r1c/bench.json
timeout 900 python tools/sweep.py --out gpurun_out/r1c/sweep.md > gpurun_out/r1c/sweep.log 2>&1
ls gpurun_out/r1c
