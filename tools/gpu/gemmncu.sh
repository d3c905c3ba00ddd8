#!/bin/bash
# One ncu --set full capture (with source) of the bin GEMM at the configs[4] shard fwd.
out=gpurun_out/${1:-gemmncu}; mkdir -p $out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:oaa_bin_gemm -c 1 -o $out/gemm_fwd python tools/prof_step.py 1 fwd 128,64,128,224,8 > $out/ncu.log 2>&1
ncu -i $out/gemm_fwd.ncu-rep --page source --csv --print-source sass > $out/src_gemm.csv 2>/dev/null
ls -la $out
