#!/bin/bash
# A/B of experiment builds: python tools/kernel_breakdown.py per library and config.
out=gpurun_out/ab; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tensor_core or fused or gemm" > $out/p.log 2>&1; echo "rc=$?" >> $out/p.log
for lib in "" $(ls -d paper_1601_06815_b200/_build_oaa_exp_* 2>/dev/null); do
  for cfg in 256,96,256,27,5 128,64,128,224,8; do
    if [ -n "$lib" ]; then export OAA_LIB=$PWD/$lib/liboaa.so; else unset OAA_LIB; fi
    echo "lib=${lib:-in-tree} cfg=$cfg $(timeout 300 python tools/kernel_breakdown.py $cfg valid 3 2>&1 | tail -1)" >> $out/ab.txt
  done
done
tail -n 2 $out/p.log; cat $out/ab.txt
