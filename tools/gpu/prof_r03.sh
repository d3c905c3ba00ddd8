#!/bin/bash
# round-3 profile set: ncu --set full of the block-size (b = 16 - n) walker / bwd_data and the
# register-accumulator bwd_filter at the N = 224 sweep points n = 3, 5, 7; launch list of the bench
out=gpurun_out/${1:-prof3}; mkdir -p $out
for n in 3 5 7; do
  timeout 900 ncu --set full --clock-control none -k regex:"oaa_walk_kernel|oaa_bwdd_kernel|oaa_bwdf_kernel|oaa_xspec" -c 5 \
    -o $out/sweep_n$n python tools/prof_step.py 1 fwd,bwd_data,bwd_filter 128,3,64,224,$n > $out/ncu_n$n.log 2>&1
  python tools/ncu_table.py $out/sweep_n$n.ncu-rep "sweep point N=224 n=$n C=3 K=64 B=128 (walker and bwd_data with b = $((16 - n)), P = 15; bwd_filter b = n$([ $n -le 5 ] && echo ', register accumulators'))" >> $out/r03_ncu_sweep.md
  rm -f $out/sweep_n$n.ncu-rep
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches_bench.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-cfg5 > $out/bench_under_ncu.log 2>&1
cat $out/r03_ncu_sweep.md
