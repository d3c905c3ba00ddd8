// oaa_tc.cuh -- tensor-core (tcgen05, sm_100a) per-frequency-bin complex channel
// contraction for layers with many channels ("genuinely dense
// contraction ... on tensor cores"; PAPER.md:15 the K·C convolutions of a layer).
//
// For every bin f the contraction Ŷ_f = Ŵ_f · X̂_f (K×C complex by C×B·T complex) is
// real-ified,
//      [Yr; Yi] (2K × N) = [[Wr, −Wi], [Wi, Wr]] (2K × 2C) · [Xr; Xi] (2C × N),
// and evaluated as D[f] = A[f] · B[f]ᵀ with A[f] = M×Kd, B[f] = N×Kd (both K-major, fp32
// in global memory).  fp32 accuracy (rel-L2 ≤ 1e-5, R9) needs 3×TF32: every
// operand is split x = hi + lo (hi = x with the low 13 mantissa bits cleared, lo = x − hi)
// and D = A_hi·B_hi + A_hi·B_lo + A_lo·B_hi accumulates in tensor memory.
//
// Kernel structure (one CTA = one 128×128 output tile of one bin, 128 threads):
//   * all threads load a 128×32 chunk of A and of B, split hi/lo and store them into shared
//     memory in the canonical no-swizzle K-major UMMA layout (8-row × 16-byte core
//     matrices; LBO = 128 B between the two K halves of an MMA, SBO = 1 KB between 8-row
//     groups), double buffered so the next chunk loads while the MMAs of this one run;
//   * one elected thread issues 4 k-steps × 3 tcgen05.mma.kind::tf32 (M=128, N=128, K=8)
//     per chunk and commits them to an mbarrier;
//   * epilogue: tcgen05.ld of the 128×128 fp32 accumulator (thread = row) → global.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace oaa {

constexpr int kTcM = 128, kTcN = 128, kTcK = 32;  // CTA tile and K chunk (fp32 elements)

struct BinGemmParams {
  const float* A;  // [F][M][Kd]
  const float* B;  // [F][N][Kd]
  float* D;        // [F][M][ldd] (row m, column n)
  int F, M, N, Kd, ldd;
  long long strideA, strideB, strideD;  // per-bin strides (elements)
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// UMMA shared-memory descriptor, K-major, no swizzle (Blackwell version 1).
__device__ __forceinline__ uint64_t umma_desc_kmajor(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version = 1 (sm_100)
  // base_offset 0, lbo_mode 0, layout_type 0 (SWIZZLE_NONE)
  return d;
}

// Instruction descriptor: D f32, A/B tf32, both K-major, M=128, N=128.
__host__ __device__ constexpr uint32_t umma_idesc_tf32(int M, int N) {
  return (1u << 4)                 // c_format = F32
         | (2u << 7)               // a_format = TF32
         | (2u << 10)              // b_format = TF32
         | (0u << 15) | (0u << 16) // K-major A and B
         | ((uint32_t)(N >> 3) << 17)
         | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void umma_tf32(uint32_t dtmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(dtmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// Split fp32 → (tf32 hi, fp32 remainder).  The tensor core reads the top 19 bits of each
// fp32 operand, so hi is exact and lo carries the next 11+ bits.
__device__ __forceinline__ void split_tf32(float x, float& hi, float& lo) {
  hi = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
  lo = x - hi;
}

// Store a 128-row × 32-element fp32 chunk (row stride ld elements in global, rows r0..)
// as hi and lo tiles in the canonical K-major no-swizzle layout:
//   byte offset of (row r, k) = (r/8)·1024 + (k/4)·128 + (r%8)·16 + (k%4)·4
// Rows ≥ nrows and columns ≥ kvalid are zero.
__device__ __forceinline__ void load_split_tile(const float* __restrict__ g, long long ld, int nrows, int kvalid,
                                                float* hi, float* lo, int tid) {
  // 128 rows × 8 chunks of 4 → 1024 float4 slots, 128 threads → 8 each
#pragma unroll
  for (int it = 0; it < 8; ++it) {
    const int slot = it * 128 + tid;
    const int r = slot >> 3, c = slot & 7;  // row, k-chunk
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (r < nrows) {
      const float* src = g + (long long)r * ld + 4 * c;
      if (4 * c + 3 < kvalid) {
        v = *reinterpret_cast<const float4*>(src);
      } else {
        if (4 * c + 0 < kvalid) v.x = src[0];
        if (4 * c + 1 < kvalid) v.y = src[1];
        if (4 * c + 2 < kvalid) v.z = src[2];
      }
    }
    float4 h, l;
    split_tf32(v.x, h.x, l.x);
    split_tf32(v.y, h.y, l.y);
    split_tf32(v.z, h.z, l.z);
    split_tf32(v.w, h.w, l.w);
    const int off = (r >> 3) * 256 + c * 32 + (r & 7) * 4;  // in floats
    *reinterpret_cast<float4*>(hi + off) = h;
    *reinterpret_cast<float4*>(lo + off) = l;
  }
}

// D[f][m][n] = Σ_k A[f][m][k] · B[f][n][k]  (3×TF32).  grid = (ceil(N/128), ceil(M/128), F)
__global__ void __launch_bounds__(128, 1) oaa_bin_gemm_kernel(const BinGemmParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // [2 buffers][A_hi, A_lo, B_hi, B_lo] × 16 KB
  float* sm = reinterpret_cast<float*>(smem_raw);
  __shared__ uint64_t mbar[2];
  __shared__ uint32_t s_tmem;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int f = blockIdx.z, m0 = blockIdx.y * kTcM, n0 = blockIdx.x * kTcN;
  const float* A = p.A + (long long)f * p.strideA + (long long)m0 * p.Kd;
  const float* Bm = p.B + (long long)f * p.strideB + (long long)n0 * p.Kd;
  const int mrows = min(kTcM, p.M - m0), nrows = min(kTcN, p.N - n0);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s_tmem;
  constexpr uint32_t idesc = umma_idesc_tf32(kTcM, kTcN);
  const int nchunks = (p.Kd + kTcK - 1) / kTcK;
  uint32_t phase[2] = {0u, 0u};
  for (int ch = 0; ch < nchunks; ++ch) {
    const int buf = ch & 1;
    float* base = sm + buf * 4 * 4096;
    // the MMAs that read this buffer two chunks ago must be done
    if (ch >= 2) {
      mbar_wait(&mbar[buf], phase[buf]);
      phase[buf] ^= 1u;
    }
    const int k0 = ch * kTcK, kvalid = min(kTcK, p.Kd - k0);
    load_split_tile(A + k0, p.Kd, mrows, kvalid, base, base + 4096, tid);
    load_split_tile(Bm + k0, p.Kd, nrows, kvalid, base + 2 * 4096, base + 3 * 4096, tid);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t a_hi = smem_u32(base), a_lo = smem_u32(base + 4096);
      const uint32_t b_hi = smem_u32(base + 2 * 4096), b_lo = smem_u32(base + 3 * 4096);
#pragma unroll
      for (int ks = 0; ks < kTcK / 8; ++ks) {  // K = 8 tf32 per MMA = 2 core-matrix columns
        const uint32_t koff = ks * 256;        // 2 × 128 B
        const uint64_t dah = umma_desc_kmajor(a_hi + koff, 128, 1024);
        const uint64_t dal = umma_desc_kmajor(a_lo + koff, 128, 1024);
        const uint64_t dbh = umma_desc_kmajor(b_hi + koff, 128, 1024);
        const uint64_t dbl = umma_desc_kmajor(b_lo + koff, 128, 1024);
        const uint32_t acc = (ch > 0 || ks > 0) ? 1u : 0u;
        umma_tf32(tmem, dal, dbh, idesc, acc);
        umma_tf32(tmem, dah, dbl, idesc, 1u);
        umma_tf32(tmem, dah, dbh, idesc, 1u);
      }
      umma_commit(&mbar[buf]);
    }
  }
  // wait for the last chunk's MMAs (all earlier ones complete in order)
  {
    const int last = (nchunks - 1) & 1;
    // each buffer's barrier has completed floor(uses) phases already consumed above
    mbar_wait(&mbar[last], phase[last]);
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // epilogue: thread tid owns accumulator row m0 + tid (TMEM lane = 32·warp + lane)
  const int row = tid;
  float* drow = p.D + (long long)f * p.strideD + (long long)(m0 + row) * p.ldd + n0;
#pragma unroll
  for (int c0 = 0; c0 < kTcN; c0 += 32) {
    float v[32];
    const uint32_t ta = tmem + ((uint32_t)(32 * warp) << 16) + c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]),
          "=f"(v[8]), "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]), "=f"(v[14]), "=f"(v[15]),
          "=f"(v[16]), "=f"(v[17]), "=f"(v[18]), "=f"(v[19]), "=f"(v[20]), "=f"(v[21]), "=f"(v[22]), "=f"(v[23]),
          "=f"(v[24]), "=f"(v[25]), "=f"(v[26]), "=f"(v[27]), "=f"(v[28]), "=f"(v[29]), "=f"(v[30]), "=f"(v[31])
        : "r"(ta));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (row < mrows) {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (c0 + j < nrows) drow[c0 + j] = v[j];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

}  // namespace oaa

#ifdef OAA_DEFINE_AUX_KERNELS
namespace oaa {
// A operand of the bin GEMM, the real-ified kernel spectra
//   Ag[f][m][kk] = [[Wr, −Wi], [Wi, Wr]]  (rows m < Co | m ≥ Co, columns kk < Ci | kk ≥ Ci),
// with W_{o,i}[f] = DFT_P(w_{o,i})[f1][f2] / P² (fwd: o = k, i = c) or of flip180(w_{k,c})
// with o = c, i = k (bwd_data).  The K padding columns (2Ci ≤ kk < Kdp) are zeroed by the
// caller.  One thread per (f, o, i), twiddles from a per-block fp64 table.
__global__ void oaa_realified_spectrum_kernel(const float* __restrict__ w, float* __restrict__ Ag, int K, int C,
                                              int n, int flip_bwd, int Kdp) {
  const int P = 2 * n - 1, H = n, F = H * P;
  const int Co = flip_bwd ? C : K, Ci = flip_bwd ? K : C;
  __shared__ double tc[16], ts[16];
  if (threadIdx.x < P) sincospi(2.0 * (double)threadIdx.x / (double)P, &ts[threadIdx.x], &tc[threadIdx.x]);
  __syncthreads();
  const long long total = (long long)F * Co * Ci;
  const double inv = 1.0 / ((double)P * (double)P);
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(t % Ci);
    const int o = (int)((t / Ci) % Co);
    const int f = (int)(t / ((long long)Ci * Co));
    const int f1 = f / P, f2 = f - (f / P) * P;
    const int k = flip_bwd ? i : o, c = flip_bwd ? o : i;
    const float* wk = w + ((size_t)k * C + c) * n * n;
    double sr = 0.0, si = 0.0;
    for (int p1 = 0; p1 < n; ++p1)
      for (int p2 = 0; p2 < n; ++p2) {
        const float v = flip_bwd ? wk[(n - 1 - p1) * n + (n - 1 - p2)] : wk[p1 * n + p2];
        const int mm = (f1 * p1 + f2 * p2) % P;
        sr += (double)v * tc[mm];
        si -= (double)v * ts[mm];
      }
    const float re = (float)(sr * inv), im = (float)(si * inv);
    float* row_r = Ag + ((long long)f * 2 * Co + o) * Kdp;
    float* row_i = row_r + (long long)Co * Kdp;
    row_r[i] = re;
    row_r[Ci + i] = -im;
    row_i[i] = im;
    row_i[Ci + i] = re;
  }
}
}  // namespace oaa
#endif
