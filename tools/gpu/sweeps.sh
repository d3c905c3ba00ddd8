#!/bin/bash
out=gpurun_out/sw; mkdir -p $out
timeout 1200 python tools/paper_sweeps.py --out $out/r02_paper_sweeps.md > $out/log.txt 2>&1; echo "rc=$?" >> $out/log.txt
timeout 1200 python tools/sweep.py --out $out/r02_sweep.md > $out/sweep_log.txt 2>&1; echo "rc=$?" >> $out/sweep_log.txt
tail -n 3 $out/log.txt $out/sweep_log.txt
