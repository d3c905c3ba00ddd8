#!/bin/bash
# bench line (driver defaults + a longer run), reference arm, launch list of the bench
out=gpurun_out/${1:-bench}; mkdir -p $out
timeout 900 python bench.py > $out/bench_default.json 2> $out/bench_default.err
timeout 900 python bench.py --steps 20 --warmup 5 > $out/bench.json 2> $out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $out/bench_ref.json 2> $out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches_bench.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-cfg5 > $out/bench_under_ncu.log 2>&1
head -c 2500 $out/bench.json
