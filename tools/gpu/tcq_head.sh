#!/bin/bash
# tensor-core-path and OaS tests + breakdowns of configs[4] shard, AlexNet and the headline
out=gpurun_out/${1:-tcqh}; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q -k "tensor_core or alexnet or sharded or config5 or fused or tcgen05 or prepared or graph or oas" > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/pytest.log
for cfg in 128,64,128,224,8 256,96,256,27,5 128,3,64,224,8; do
  timeout 600 python tools/kernel_breakdown.py $cfg valid 3 >> $out/bd.json 2>&1
done
tail -3 $out/pytest.log; cat $out/bd.json
