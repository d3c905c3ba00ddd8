#!/bin/bash
# round-2 profile set: headline traffic + ncu --set full of the headline kernels, tensor-core path
# kernels at configs[4] shard / configs[3], the BASELINE sweep.
out=gpurun_out/${1:-prof}; mkdir -p $out
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
  --log-file $out/traffic_headline.csv python tools/prof_step.py 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"oaa_walk_kernel|oaa_bwdd_kernel|oaa_bwdf_kernel|oaa_xspec|finalize|spectrum" -c 7 \
  -o $out/headline_full python tools/prof_step.py 1 > $out/ncu_headline.log 2>&1
timeout 1200 ncu --set full --clock-control none -k regex:"oaa_bin_gemm|oaa_walk_kernel|oaa_tile_spectra|oaa_filter_spectra" -c 9 \
  -o $out/tc_shard python tools/prof_step.py 1 fwd,bwd_data,bwd_filter 128,64,128,224,8 > $out/ncu_tc.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"oaa_bin_gemm" -c 3 \
  -o $out/tc_alexnet python tools/prof_step.py 1 fwd,bwd_data,bwd_filter 256,96,256,27,5 > $out/ncu_alex.log 2>&1
timeout 1800 python tools/sweep.py --out $out/r02_sweep.md > $out/sweep.log 2>&1
ls -la $out
python tools/traffic_json.py $out/traffic_headline.csv > $out/r02_traffic.json
python tools/ncu_table.py $out/headline_full.ncu-rep "Headline step kernels (N=224 n=8 C=3 K=64 B=128; ncu --set full, --clock-control none, serialized)" > $out/r02_ncu_kernels.md
python tools/ncu_table.py $out/tc_shard.ncu-rep "configs[4] per-GPU shard (N=224 n=8 C=64 K=128 B=128), tensor-core path, one pass each of fwd, bwd_data, bwd_filter" >> $out/r02_ncu_kernels.md
python tools/ncu_table.py $out/tc_alexnet.ncu-rep "AlexNet-like (N=27 n=5 C=96 K=256 B=256) bin GEMMs" >> $out/r02_ncu_kernels.md
rm -f $out/tc_shard.ncu-rep $out/tc_alexnet.ncu-rep
du -sh $out
