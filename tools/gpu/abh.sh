#!/bin/bash
# A/B of experiment builds on the headline (and extra configs given as arguments): kernel breakdown per library.
out=gpurun_out/${1:-abh}; shift; mkdir -p $out
cfgs="${@:-128,3,64,224,8}"
for lib in "" $(ls -d paper_1601_06815_b200/_build_oaa_exp_* 2>/dev/null); do
  for cfg in $cfgs; do
    if [ -n "$lib" ]; then export OAA_LIB=$PWD/$lib/liboaa.so; else unset OAA_LIB; fi
    echo "lib=${lib:-in-tree} cfg=$cfg $(timeout 300 python tools/kernel_breakdown.py $cfg valid 5 2>&1 | tail -1)" >> $out/ab.txt
  done
done
cat $out/ab.txt
