#!/bin/bash
# GPU suite, headline kernel breakdown, compute-sanitizer memcheck / racecheck / synccheck (tools/sanitize_cases.py) and the toy-library check (tools/sanity_lib.py).
out=gpurun_out/${1:-tma}; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -x -q > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/pytest.log
timeout 300 python tools/kernel_breakdown.py 128,3,64,224,8 valid 5 > $out/bd.json 2>&1
timeout 300 compute-sanitizer --tool memcheck python tools/sanity_lib.py > $out/sanitizer_minimal_lib.txt 2>&1
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_cases.py > $out/sanitizer_memcheck.txt 2>&1; echo "exit=$?" >> $out/sanitizer_memcheck.txt
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_cases.py > $out/sanitizer_racecheck.txt 2>&1; echo "exit=$?" >> $out/sanitizer_racecheck.txt
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_cases.py > $out/sanitizer_synccheck.txt 2>&1; echo "exit=$?" >> $out/sanitizer_synccheck.txt
tail -3 $out/pytest.log; cat $out/bd.json; for f in $out/sanitizer_*.txt; do tail -n 3 $f; done
