#!/bin/bash
# tensor-core path: parity tests (small + full size) and the per-kernel breakdown at configs[3], configs[4] shard
out=gpurun_out/${1:-tcq}; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q -k "tensor_core or alexnet or sharded or config5 or fused or tcgen05 or prepared or graph" > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/pytest.log
timeout 600 python tools/kernel_breakdown.py 128,64,128,224,8 valid 3 > $out/bd.json 2>&1
timeout 600 python tools/kernel_breakdown.py 256,96,256,27,5 valid 3 >> $out/bd.json 2>&1
tail -3 $out/pytest.log; cat $out/bd.json
