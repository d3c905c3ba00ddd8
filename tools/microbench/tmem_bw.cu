// Microbenchmark: tcgen05.ld / tcgen05.st throughput (32x32b shape: each thread owns a
// TMEM lane and reads/writes consecutive 32-bit columns).  Informs whether per-lane
// spectra can live in TMEM instead of registers.  Not product code.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define ITERS 2048
__device__ __forceinline__ void tld16(uint32_t taddr, float* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]),
                 "=f"(v[8]), "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]), "=f"(v[14]), "=f"(v[15])
               : "r"(taddr));
}
__device__ __forceinline__ void tst16(uint32_t taddr, const float* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
               :: "r"(taddr), "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]),
                 "f"(v[8]), "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]));
}
template <int MODE>  // 0: ld only, 1: st only, 2: ld+fma+st
__global__ void __launch_bounds__(256, 1) tmem_kernel(float* out, int ncols_per_thread) {
  __shared__ uint32_t s_taddr;
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"((uint32_t)__cvta_generic_to_shared(&s_taddr)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = s_taddr;
  const uint32_t lane_base = (uint32_t)(32 * (warp % 4)) << 16;
  const uint32_t col0 = (warp / 4) * 256;  // 8 warps: two per quadrant, 256 columns each
  float acc[16];
  for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x + i;
  for (int it = 0; it < ITERS; ++it) {
    for (int c = 0; c < ncols_per_thread; c += 16) {
      const uint32_t ta = base + lane_base + col0 + c;
      if (MODE == 0) {
        float v[16];
        tld16(ta, v);
        asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] += v[i];
      } else if (MODE == 1) {
        tst16(ta, acc);
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] += 1.0f;
      } else {
        float v[16];
        tld16(ta, v);
        asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = fmaf(v[i], 0.999f, acc[i]);
        tst16(ta, v);
      }
    }
  }
  asm volatile("tcgen05.wait::st.sync.aligned;");
  float s = 0;
  for (int i = 0; i < 16; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(base));
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out; cudaMalloc(&out, 1 << 24);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int ncols = 128;
  auto run = [&](const char* name, auto k) {
    k<<<sms, 256>>>(out, ncols); cudaDeviceSynchronize();
    cudaEventRecord(a); k<<<sms, 256>>>(out, ncols); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double bytes = (double)sms * 256 * ITERS * ncols * 4;
    printf("%-8s %8.3f ms  %8.1f GB/s total  %6.1f B/clk/SM @1.9GHz   err=%s\n", name, ms, bytes / ms / 1e6,
           bytes / (ms * 1e-3) / sms / 1.9e9, cudaGetErrorString(cudaGetLastError()));
  };
  run("ld", tmem_kernel<0>);
  run("st", tmem_kernel<1>);
  run("ld+st", tmem_kernel<2>);
  return 0;
}
