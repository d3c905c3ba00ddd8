// Microbenchmark: the two compute roofline denominators of SURVEY.md §8(d) that
// MEASURED_PEAKS.json does not carry, measured on the B200 itself (not product code):
//   * fp32 FFMA issue rate (all SMs, 64 warps per SM, 8 independent chains per thread);
//   * tcgen05.mma kind::tf32 dense throughput (one CTA per SM, M=128 N=256 K=8, the
//     shape of the product's bin GEMM, operands resident in shared memory, one thread
//     issuing back-to-back MMAs into two alternating TMEM accumulators);
//   * tcgen05.mma kind::f16 (bf16) with the same harness, as a cross-check of the harness
//     against the driver-measured cuBLAS bf16 peak in MEASURED_PEAKS.json.
// Prints one JSON line.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 peaks.cu
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>

#define FF_ITERS 8192
__global__ void __launch_bounds__(512) ffma_reg(float* out, float a, float b) {
  float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < FF_ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b);
      x4 = fmaf(x4, a, b); x5 = fmaf(x5, a, b); x6 = fmaf(x6, a, b); x7 = fmaf(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_kmajor(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
// idesc: D f32; a/b format 2 = TF32 (kind::tf32) or 1 = BF16 (kind::f16); K-major; N>>3, M>>4
__host__ __device__ constexpr uint32_t idesc(int fmt, int M, int N) {
  return (1u << 4) | ((uint32_t)fmt << 7) | ((uint32_t)fmt << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

template <bool TF32>
__global__ void __launch_bounds__(128, 1) mma_peak(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) unsigned char sm[];  // A 128 rows × 32 B | B 256 rows × 32 B (one K step)
  __shared__ uint64_t bar;
  __shared__ uint32_t s_tmem;
  const int tid = threadIdx.x;
  for (int i = tid; i < (128 + 256) * 32 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.01f * (float)(i % 13) - 0.06f;
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0) {
    const uint32_t a = smem_u32(sm), b = a + 128 * 32;
    // one K step = 32 bytes per row = two 16-byte core-matrix columns (LBO 128 B would be
    // for a 2-column block stored column-major by 8×16 B core matrices; SBO 256 B per 8 rows)
    const uint64_t da = desc_kmajor(a, 128, 256), db = desc_kmajor(b, 128, 256);
    const uint32_t id = idesc(TF32 ? 2 : 1, 128, 256);
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t acc = s_tmem + (i & 1) * 256;
      if (TF32)
        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}"
                     ::"r"(acc), "l"(da), "l"(db), "r"(id), "r"(1) : "memory");
      else
        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}"
                     ::"r"(acc), "l"(da), "l"(db), "r"(id), "r"(1) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                 : "memory");
    asm volatile(
        "{\n .reg .pred p;\n W:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W;\n}" ::"r"(
            smem_u32(&bar))
        : "memory");
    cycles[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(s_tmem));
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  const int sms = p.multiProcessorCount;
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  float* out;
  cudaMalloc(&out, 1 << 26);
  unsigned long long* cyc;
  cudaMalloc(&cyc, sizeof(unsigned long long) * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto best_ms = [&](auto launch) {
    launch();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 7; ++r) {
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      best = ms < best ? ms : best;
    }
    return best;
  };
  // FFMA: 4 CTAs × 512 threads per SM
  const int fb = sms * 4, ft = 512;
  const double ffma_flops = 2.0 * fb * ft * FF_ITERS * 32;
  const float ffma_ms = best_ms([&] { ffma_reg<<<fb, ft>>>(out, 0.999f, 0.001f); });
  // tcgen05 tf32 / bf16, M=128 N=256 K=8 (tf32) or K=16 (bf16) per instruction
  const int iters = 1 << 16;
  const size_t smem = (128 + 256) * 32;
  const float tf_ms = best_ms([&] { mma_peak<true><<<sms, 128, smem>>>(iters, cyc); });
  const float bf_ms = best_ms([&] { mma_peak<false><<<sms, 128, smem>>>(iters, cyc); });
  const double tf_flops = 2.0 * 128 * 256 * 8 * (double)iters * sms;
  const double bf_flops = 2.0 * 128 * 256 * 16 * (double)iters * sms;
  cudaError_t e = cudaDeviceSynchronize();
  printf("{\"device\": \"%s\", \"sms\": %d, \"clock_khz_attr\": %d, "
         "\"ffma_tflops\": %.2f, \"ffma_ms\": %.4f, "
         "\"tcgen05_tf32_tflops\": %.1f, \"tf32_ms\": %.4f, "
         "\"tcgen05_bf16_tflops\": %.1f, \"bf16_ms\": %.4f, \"err\": \"%s\"}\n",
         p.name, sms, clk_khz, ffma_flops / ffma_ms / 1e9, ffma_ms, tf_flops / tf_ms / 1e9, tf_ms,
         bf_flops / bf_ms / 1e9, bf_ms, cudaGetErrorString(e));
  return e == cudaSuccess ? 0 : 1;
}
