#!/bin/bash
# A/B of experiment builds (python -m paper_1601_06815_b200.build -DOAA_EXP_…) by kernel breakdown,
# interleaved over ROUNDS rounds (default 2) so that drift hits every library alike.
# usage: abh.sh NAME [cfg ...]   cfg = B,C,K,N,n   (default: the headline)
out=gpurun_out/${1:-abh}; shift; mkdir -p $out
cfgs="${@:-128,3,64,224,8}"
for r in $(seq 1 ${ROUNDS:-2}); do
  for lib in "" $(ls -d paper_1601_06815_b200/_build_oaa_exp_* 2>/dev/null); do
    for cfg in $cfgs; do
      if [ -n "$lib" ]; then export OAA_LIB=$PWD/$lib/liboaa.so; else unset OAA_LIB; fi
      echo "r=$r lib=${lib:-in-tree} cfg=$cfg $(timeout 300 python tools/kernel_breakdown.py $cfg valid 5 2>&1 | tail -1)" >> $out/ab.txt
    done
  done
done
cat $out/ab.txt
