#!/bin/bash
# Full GPU check: host memory, GPU test suite (timed), smoke, bench (1 GPU).
out=gpurun_out/${1:-check}; mkdir -p $out
free -g > $out/free.txt
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > $out/bench.json 2> $out/bench.err; echo "bench rc=$?" >> $out/bench.err
tail -5 $out/pytest.log; tail -3 $out/smoke.log; cat $out/bench.json | head -c 3000
