#!/bin/bash
# compute-sanitizer passes, the ncu launch list of the bench command, per-kernel DRAM traffic
# of the headline step, and one --set full capture of the top kernels.
out=gpurun_out/prof; mkdir -p $out
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py > $out/sanitizer_$tool.txt 2>&1
  echo "exit=$?" >> $out/sanitizer_$tool.txt
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches_bench.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-cfg5 > $out/bench_under_ncu.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
  --log-file $out/traffic_headline.csv python tools/prof_step.py 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"oaa_walk_kernel|oaa_bwdd_kernel|oaa_bwdf_kernel|oaa_xspec" -c 5 \
  -o $out/headline_full python tools/prof_step.py 1 > $out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:oaa_bin_gemm -s 1 -c 2 -o $out/gemm_alexnet python tools/prof_step.py 2 fwd 256,96,256,27,5 > /dev/null 2>&1
tail -n 2 $out/sanitizer_*.txt; ls -la $out
