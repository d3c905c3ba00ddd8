#!/bin/bash
out=gpurun_out/bd; mkdir -p $out
for cfg in 128,3,64,224,8 256,96,256,27,5 128,64,128,224,8 1024,64,128,224,8; do
  timeout 300 python tools/kernel_breakdown.py $cfg valid 3 >> $out/bd.jsonl 2>&1
done
cat $out/bd.jsonl
