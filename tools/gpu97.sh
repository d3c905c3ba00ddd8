mkdir -p gpurun_out/r1d
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:oaa_bin_gemm -s 1 -c 1 -o gpurun_out/r1d/gemm python tools/prof_step.py 2 fwd 256,96,256,27,5 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:oaa_filter_spectra -s 0 -c 1 -o gpurun_out/r1d/fspec python tools/prof_step.py 1 bwd_filter 128,64,128,224,8 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1d/shard.csv python tools/prof_step.py 1 fwd,bwd_data,bwd_filter 128,64,128,224,8 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1d/alex.csv python tools/prof_step.py 1 fwd,bwd_data,bwd_filter 256,96,256,27,5 > /dev/null 2>&1
timeout 600 python bench.py 2>&1 | tail -1 > gpurun_out/r1d/bench.json
timeout 900 python tools/sweep.py --out gpurun_out/r1d/sweep.md > gpurun_out/r1d/sweep.log 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
ls gpurun_out/r1d
