#!/bin/bash
# GPU suite + per-kernel breakdown at the sweep's small sizes and n = 3/5/7 at N = 224.
out=gpurun_out/${1:-small}; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -x -q > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/pytest.log
for cfg in 128,3,64,16,8 128,3,64,32,8 128,3,64,64,8 128,3,64,16,3 128,3,64,64,3 128,3,64,224,3 128,3,64,224,5 128,3,64,224,7 128,3,64,224,8; do
  timeout 300 python tools/kernel_breakdown.py $cfg valid 5 >> $out/bd.jsonl 2>&1
done
tail -3 $out/pytest.log; cat $out/bd.jsonl
