mkdir -p gpurun_out/r1e
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1e/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1e/alex.csv python tools/prof_step.py 1 fwd,bwd_data,bwd_filter 256,96,256,27,5 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1e/shard.csv python tools/prof_step.py 1 fwd,bwd_data,bwd_filter 128,64,128,224,8 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:oaa_bin_gemm -s 1 -c 1 -o gpurun_out/r1e/gemm python tools/prof_step.py 1 fwd,bwd_data 128,64,128,224,8 > /dev/null 2>&1
timeout 600 python bench.py 2>&1 | tail -1 > gpurun_out/r1e/bench.json
timeout 900 python tools/sweep.py --out gpurun_out/r1e/sweep.md > gpurun_out/r1e/sweep.log 2>&1
ls gpurun_out/r1e
