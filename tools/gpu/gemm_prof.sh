#!/bin/bash
out=gpurun_out/gp; mkdir -p $out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:oaa_bin_gemm -s 1 -c 1 -o $out/gemm_shard_fwd python tools/prof_step.py 2 fwd 128,64,128,224,8 > $out/l1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:oaa_walk_kernel -s 1 -c 1 -o $out/walkload_shard_fwd python tools/prof_step.py 2 fwd 128,64,128,224,8 > $out/l2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:oaa_tile_spectra -s 1 -c 1 -o $out/tilespec_shard_fwd python tools/prof_step.py 2 fwd 128,64,128,224,8 > $out/l3.log 2>&1
cat > /tmp/sanity_min.cu <<'CU'
#include <cstdio>
__global__ void k(float* p) { p[threadIdx.x] = 1.f; }
int main() { float* p; cudaMalloc(&p, 1024); k<<<1, 32>>>(p); printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize())); }
CU
nvcc -gencode arch=compute_100a,code=sm_100a /tmp/sanity_min.cu -o /tmp/sanity_min && compute-sanitizer --tool memcheck /tmp/sanity_min > $out/sanitizer_minimal.txt 2>&1
ls -la $out; cat $out/sanitizer_minimal.txt
