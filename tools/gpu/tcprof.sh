#!/bin/bash
# ncu --set full of each tensor-core-path kernel at the configs[4] per-GPU shard (B=128, C=64, K=128).
out=gpurun_out/${1:-tcprof}; mkdir -p $out
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"oaa_bin_gemm|oaa_walk_kernel|oaa_tile_spectra|oaa_filter_spectra" -c 8 \
  -o $out/tc_shard python tools/prof_step.py 1 fwd,bwd_data,bwd_filter 128,64,128,224,8 > $out/ncu.log 2>&1
timeout 600 python tools/kernel_breakdown.py 128,64,128,224,8 valid 3 > $out/bd.json 2>&1
timeout 600 python tools/kernel_breakdown.py 256,96,256,27,5 valid 3 >> $out/bd.json 2>&1
tail -3 $out/ncu.log; cat $out/bd.json
