#!/bin/bash
# One ncu --set full capture (with source) of each headline kernel, for tools/sass_hot.py.
out=gpurun_out/${1:-hot}; mkdir -p $out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"oaa_walk_kernel|oaa_bwdd_kernel|oaa_bwdf_kernel" -c 3 \
  -o $out/headline_full python tools/prof_step.py 1 > $out/ncu_full.log 2>&1
for k in walk bwdd bwdf; do
  ncu -i $out/headline_full.ncu-rep -k regex:oaa_${k}_kernel --page source --csv --print-source sass > $out/src_$k.csv 2>/dev/null
done
ls -la $out
