#!/bin/bash
# forward walker with blocks b != n: parity (walker tests, full-size sweep points) + breakdowns of the sweep
out=gpurun_out/${1:-bsz}; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -x -q -k "walker_block_size or small_grid or largest or prepared or random or sweep_point or headline or config1 or graph" > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/pytest.log
for N in 224 128 64 32; do for n in 3 5 7 8; do
  timeout 300 python tools/kernel_breakdown.py 128,3,64,$N,$n valid 5 >> $out/bd.json 2>&1
done; done
tail -3 $out/pytest.log
