#!/bin/bash
# Round-end style check: full GPU suite, smoke, bench (1 GPU), sweeps.
out=gpurun_out/${1:-full}; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -x -q --durations=10 > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $out/bench.json 2> $out/bench.err; echo "bench rc=$?" >> $out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $out/bench_ref.json 2> $out/bench_ref.err
timeout 1800 python tools/paper_sweeps.py --out $out/r02_paper_sweeps.md > $out/sweeps.log 2>&1
timeout 1800 python tools/sweep.py --out $out/r02_sweep.md > $out/sweep.log 2>&1
tail -n 4 $out/pytest.log; tail -n 3 $out/smoke.log; head -c 1500 $out/bench.json
