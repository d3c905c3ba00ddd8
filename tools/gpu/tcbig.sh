#!/bin/bash
# tensor-core path with blocks b = 16 - n: parity + interleaved A/B against -DOAA_EXP_TC_SMALLB
out=gpurun_out/${1:-tcbig}; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -x -q -k "tensor_core or fused or alexnet or prepared or sharded or config5 or random or block_size" > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/pytest.log
ROUNDS=2 bash tools/gpu/abh.sh ${1:-tcbig}/ab 256,96,256,27,5 128,32,64,56,3 128,32,64,64,7 > /dev/null 2>&1
tail -3 $out/pytest.log
