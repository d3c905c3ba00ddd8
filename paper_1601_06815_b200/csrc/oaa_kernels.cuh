// oaa_kernels.cuh -- shared helpers and the first-generation fused kernels of the OaA layer.
//
// Where the hot path runs: the forward walker (oaa_walk.cuh), bwd_data
// (oaa_bwdd.cuh), bwd_filter (oaa_bwdf.cuh) for small channel counts; the tcgen05 bin GEMM
// (oaa_tc.cuh) with the operand producers below for C, K ≥ 16.  The engines in this file
// (oaa_engine_kernel S1/S2, oaa_engine_s1t_kernel, oaa_bwd_filter_kernel) cover the shapes
// those kernels do not (e.g. 5 ≤ C ≤ 15 with small K, or a tile row needing more than 8
// chunk warps); oaa_spectrum_kernel and oaa_filter_finalize_kernel are used by all paths.
//
// Notation: input blocks are n×n, transforms are P×P with
// P = 2n−1, the half spectrum keeps rows f1 ∈ [0,H), H = n, and all
// columns f2 ∈ [0,P) (stored as P2 = (P+1)/2 pairs, the last one zero-padded).  A
// "work item" is one tile row (b, t1) of one image.
//
//  * oaa_engine_kernel<n, CR, S1>: forward and bwd_data
//    -- tile, pad, 2-D DFT, per-bin channel contraction, inverse DFT, overlap-add, crop --
//    in ONE pass.  The item's input rows are staged in shared memory (cp.async, zero
//    padded); stage-A lanes own (tile t2, spectrum row f1); stage-B lanes own one output
//    column.  Horizontal overlap (n−1 columns) is resolved inside stage B by summing the
//    two contributing block columns BEFORE the last inverse transform (linearity);
//    vertical overlap (n−1 rows) is a read-modify-write of the previous tile row's
//    partial rows, ordered by a per-item release flag and deferred by two output
//    channels so the predecessor is normally already past it.
//      S1 (input-stationary): the input spectra of ≤ CR channels live in registers and
//         every output channel is contracted + inverse-transformed in turn.
//      S2 (output-stationary): ≤ CR output-channel accumulators live in registers and
//         every input channel is transformed + contracted into them.
//  * oaa_bwd_filter_kernel<n, CR>: weight gradient: per dy block s the
//    (2n−1)² x-window spectrum Ξ̂ and the block spectrum Ĝ, dŴ += conj(Ĝ)·Ξ̂; lanes own
//    (k, f1) and accumulate over a static, deterministic slice of the batch.
//  * oaa_filter_finalize_kernel: fixed-order fp64 sum of the per-CTA partial spectra,
//    inverse DFT, lag read-out dw[k,c,u,v] = r[n−1−u, n−1−v].
//  * oaa_spectrum_kernel: kernel spectra Ŵ (or of flip180(w) for bwd_data), scaled by
//    1/P² (the inverse transform's normalisation), in fp64 → fp32.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "dft.cuh"

namespace oaa {

constexpr int kMaxThreads = 256;  // CTA size cap: max(T·n, Ro) ≤ 256 ⇒ N ≲ 250

// Compile-time stride (in float2) of the tile index t2 in the shared Q buffer
// Q[f1][p2][t2]: ≥ the largest T = kMaxThreads/n, and ≡ 16/n (mod 16) so stage-A
// stores (lanes = (t2, f1)) and stage-B loads (lanes = consecutive output columns) of
// 64-bit words are (near) bank-conflict free.  Shared by host planning and kernels.
__host__ __device__ constexpr int q_stride(int n) {
  int target = (16 / n) % 16;
  if (target == 0) target = 16 % 16;
  int ts = (kMaxThreads + n - 1) / n + 1;  // + ≥1 always-zero column (see col_geo)
  while ((ts % 16) != target) ++ts;
  return ts;
}

struct EngineParams {
  const float* in;      // [B][Cin][R][R]
  const float4* spec;   // [Cloop][Cinner][P2][H] (f2 pairs; S1: loop=cout, S2: loop=cin)
  float* out;           // [B][Cout][Ro][Ro]
  int* flags;           // [B*T] progress of each work item (# output channels stored)
  int* counter;         // dynamic work-item counter
  int B, Cin, Cout, R, T, Ro, off, TS, BW, num_items;
  int ncomp;            // compute threads; a trailing extra warp (if any) only publishes flags
  int CIG;              // S2: input channels staged per barrier
  // tensor-core path (LY engine): Ŷ = D[f][m][bt] from the bin GEMM, items of the batch
  // chunk starting at image b0 (item = (b − b0)·T + t1), BTc = tiles in the chunk
  const float* D;
  int BTc, b0;
};

struct FilterParams {
  const float* x;       // [B][C][N][N]
  const float* dy;      // [B][K][M][M]
  float2* partial;      // [G][K][C][P][H]
  int B, C, K, N, M, off, Td, G, KG, TCH, XW, DW;
};

// ------------------------------------------------------------ memory helpers
__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Release fence at GPU scope: prior writes of this thread become visible device-wide
// before its later writes (MEMBAR.ALL.GPU; unlike fence_release() it is not SC and does
// not invalidate L1).
__device__ __forceinline__ void fence_release() { asm volatile("fence.release.gpu;" ::: "memory"); }
__device__ __forceinline__ void st_release(int* p, int v) {
#ifdef OAA_EXP_RELAXED_PUBLISH
  asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
#else
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
#endif
}
__device__ __forceinline__ void cp_async4(float* smem, const float* gmem, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(s), "l"(gmem),
               "r"(valid ? 4 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// ------------------------------------------------------------ mbarrier / bulk copy
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

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
// Same wait, but each try suspends the thread (up to the hint, in ns) until the phase
// completes instead of returning at once: for the role warps of the tensor-core pipeline,
// whose busy spinning (BRA / YIELD / SYNCS) otherwise takes issue slots from the warps doing
// the work.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(1000000u)
      : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// 1-D bulk copy global → shared (TMA engine), completion counted on `bar` in bytes.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
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

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// Stage rows [r0, r0+nrows) × cols [c0, c0+ncols) of an R×R plane into smem rows of
// stride `ld` (zero outside the plane: the zero-filled edge blocks of PAPER.md:18).
// Threads own columns (no integer division); rows whose start is 16-byte aligned and
// whose column range is a multiple of 4 go through 16-byte cp.async.
__device__ __forceinline__ void stage_rows(float* dst, int ld, const float* __restrict__ plane,
                                           int R, int r0, int nrows, int c0, int ncols, int tid,
                                           int nthr) {
  if (((R | c0 | ncols | ld) & 3) == 0) {
    for (int g = tid; g < (ncols >> 2); g += nthr) {
      const int q = c0 + 4 * g;
      const bool qok = q >= 0 && q < R;  // groups are entirely in or out (R % 4 == 0)
      for (int rr = 0; rr < nrows; ++rr) {
        const int r = r0 + rr;
        const bool ok = qok && r >= 0 && r < R;
        const unsigned sa = (unsigned)__cvta_generic_to_shared(dst + rr * ld + 4 * g);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa),
                     "l"(ok ? plane + (size_t)r * R + q : plane), "r"(ok ? 16 : 0)
                     : "memory");
      }
    }
  } else {
    for (int cc = tid; cc < ncols; cc += nthr) {
      const int q = c0 + cc;
      const bool qok = q >= 0 && q < R;
      const float* src = plane + (size_t)r0 * R + q;  // only dereferenced when in range
      float* d = dst + cc;
      for (int rr = 0; rr < nrows; ++rr) {
        const int r = r0 + rr;
        const bool ok = qok && r >= 0 && r < R;
        cp_async4(d, ok ? src : plane, ok);
        src += R;
        d += ld;
      }
    }
  }
}

// Read one n×n block from staged rows (row stride ld, block column origin c).
template <int NN>
__device__ __forceinline__ void read_block(const float* src, int ld, int c, float (&z)[NN][NN]) {
#pragma unroll
  for (int p1 = 0; p1 < NN; ++p1) {
    if constexpr (NN % 4 == 0) {
#pragma unroll
      for (int q = 0; q < NN; q += 4) {
        const float4 v = *reinterpret_cast<const float4*>(src + p1 * ld + c + q);
        z[p1][q] = v.x; z[p1][q + 1] = v.y; z[p1][q + 2] = v.z; z[p1][q + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int q = 0; q < NN; ++q) z[p1][q] = src[p1 * ld + c + q];
    }
  }
}

// Forward DFT of one zero-padded n×n block for ONE spectrum row f1 (the lane's):
//   X[f2] = Σ_{p2<n} ( Σ_{p1<n} z[p1][p2]·e^{−iθ f1 p1} ) e^{−iθ f2 p2},  θ = 2π/P.
// The column stage uses the lane's runtime twiddles (cf, sf); the row stage is a pruned
// compile-time codelet (inputs n..P−1 are the zero padding).
template <int NN>
__device__ __forceinline__ void block_row_spectrum(const float (&z)[NN][NN], const float (&cf)[NN],
                                                   const float (&sf)[NN], float (&xr)[2 * NN - 1],
                                                   float (&xi)[2 * NN - 1]) {
  constexpr int P = 2 * NN - 1;
  float rr[P], ri[P];
#pragma unroll
  for (int p2 = 0; p2 < NN; ++p2) {
    float a = z[0][p2], b = 0.f;  // p1 = 0 twiddle is 1
#pragma unroll
    for (int p1 = 1; p1 < NN; ++p1) {
      a = fmaf(z[p1][p2], cf[p1], a);
      b = fmaf(-z[p1][p2], sf[p1], b);
    }
    rr[p2] = a;
    ri[p2] = b;
  }
#pragma unroll
  for (int p2 = NN; p2 < P; ++p2) { rr[p2] = 0.f; ri[p2] = 0.f; }
  dft<P, -1, lead_mask(NN)>(rr, ri, xr, xi);
}

// Same as block_row_spectrum, reading the block row by row from staged shared memory
// (row stride ld, block column origin c) so the n×n block is never held in registers.
template <int NN, int P = 2 * NN - 1>
__device__ __forceinline__ void block_row_spectrum_smem(const float* src, int ld, int c, const float (&cf)[NN],
                                                        const float (&sf)[NN], float (&xr)[P], float (&xi)[P]) {
  float rr[P], ri[P];
#pragma unroll
  for (int p1 = 0; p1 < NN; ++p1) {
    float z[NN];
    if constexpr (NN % 4 == 0) {
#pragma unroll
      for (int q = 0; q < NN; q += 4) {
        const float4 v = *reinterpret_cast<const float4*>(src + p1 * ld + c + q);
        z[q] = v.x; z[q + 1] = v.y; z[q + 2] = v.z; z[q + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int q = 0; q < NN; ++q) z[q] = src[p1 * ld + c + q];
    }
#pragma unroll
    for (int p2 = 0; p2 < NN; ++p2) {
      if (p1 == 0) { rr[p2] = z[p2]; ri[p2] = 0.f; }
      else {
        rr[p2] = fmaf(z[p2], cf[p1], rr[p2]);
        ri[p2] = fmaf(-z[p2], sf[p1], ri[p2]);
      }
    }
  }
#pragma unroll
  for (int p2 = NN; p2 < P; ++p2) { rr[p2] = 0.f; ri[p2] = 0.f; }
  dft<P, -1, lead_mask(NN)>(rr, ri, xr, xi);
}

// Stage A tail: inverse DFT along f2 of one spectrum row and store it, transposed, to
// the shared Q buffer  Q[f1][p2][t2]  (complex, float2).
template <int NN>
__device__ __forceinline__ void stage_a_store(const float (&yr)[2 * NN - 1], const float (&yi)[2 * NN - 1],
                                              float2* __restrict__ Qlane) {
  constexpr int P = 2 * NN - 1, TS = q_stride(NN);
  float qr[P], qi[P];
  dft<P, +1>(yr, yi, qr, qi);
#pragma unroll
  for (int p2 = 0; p2 < P; ++p2) Qlane[p2 * TS] = make_float2(qr[p2], qi[p2]);
}

// Stage-B lane geometry for output column J (Full-frame coordinate): the two block
// columns that land on it -- block tA at p2 = pA and block tA−1 at p2 = pA + n -- as
// float2 offsets into a Q buffer, with validity flags.
// An absent contributor reads column T of the Q buffer, which is kept zero
// (zero_q_tail), so the loads need no predicates.
struct ColGeo {
  int offA, offB;
};
template <int NN>
__device__ __forceinline__ ColGeo col_geo(int J, int T) {
  constexpr int TS = q_stride(NN);
  const int tA = J / NN, pA = J - tA * NN;
  ColGeo g;
  g.offA = (tA < T) ? pA * TS + tA : pA * TS + T;
  g.offB = (tA >= 1 && pA <= NN - 2) ? (pA + NN) * TS + tA - 1 : pA * TS + T;
  return g;
}
// Zero the unused tile columns [T, TS) of both Q buffers (stage A never writes them
// with non-zero data).
template <int NN>
__device__ __forceinline__ void zero_q_tail(float2* Qs, int qsz, int T, int tid, int nthr) {
  constexpr int P = 2 * NN - 1, H = NN, TS = q_stride(NN);
  const int w = TS - T, tot = 2 * H * P * w;
  for (int e = tid; e < tot; e += nthr) {
    const int c = e % w, row = e / w;  // row = buf·H·P + f1·P + p2
    const int buf = row / (H * P), rr = row - buf * (H * P);
    Qs[buf * qsz + rr * TS + T + c] = make_float2(0.f, 0.f);
  }
}

// Sum the two block columns and apply the Hermitian inverse along f1 (c2r): y[p1] is
// block row p1 of this tile row in output column J.
template <int NN>
__device__ __forceinline__ void stage_b_column(const float2* __restrict__ Q, const ColGeo& g,
                                               float (&y)[2 * NN - 1]) {
  constexpr int P = 2 * NN - 1, H = NN, TS = q_stride(NN);
  float zr[H], zi[H];
  const float2* qa = Q + g.offA;
  const float2* qb = Q + g.offB;
#pragma unroll
  for (int f1 = 0; f1 < H; ++f1) {
    const float2 a = qa[f1 * P * TS];
    const float2 b = qb[f1 * P * TS];
    zr[f1] = a.x + b.x;
    zi[f1] = a.y + b.y;
  }
  c2r_half<P>(zr, zi, y);
}

#ifndef OAA_RING_DEPTH
#define OAA_RING_DEPTH 12
#endif
#ifndef OAA_PUBLISH_EVERY
#define OAA_PUBLISH_EVERY 8
#endif
constexpr int kRingDepth = OAA_RING_DEPTH;      // deferred output channels per stage-B lane (smem ring)
constexpr int kPublishEvery = OAA_PUBLISH_EVERY;  // progress-flag granularity (output channels)
static_assert(kRingDepth > kPublishEvery, "ring must cover the publication lag");

// Wait (one lane per warp polls) until the predecessor item published ≥ need channels.
// `seen` caches the last observed value (warp-uniform) and `inflight` is a value loaded
// one iteration earlier, so in the steady state no poll latency is exposed.  The data
// that follows is read with ld.global.cg (L2, the point of coherence), so no L1
// invalidation (acquire / fence) is needed on this path.
__device__ __forceinline__ void wait_flag(const int* flag, int need, int lane, int leader,
                                          unsigned mask, int& seen, int inflight) {
#ifdef OAA_EXP_NO_WAIT
  return;
#endif
  if (seen >= need) return;
  seen = max(seen, __shfl_sync(mask, inflight, leader));
  while (seen < need) {
    int v = 0;
    if (lane == leader) {
      v = ld_relaxed(flag);
      if (v < need) __nanosleep(64);
    }
    seen = __shfl_sync(mask, v, leader);
  }
}

// ------------------------------------------------------------------ engine
// Shared memory: Q[2][H][P][TS] (+1 zero slot each) float2 | spectra[NSB][Cinner][P2][H]
// float4 | staged input rows [S1: Cin | S2: 2][n][BW] floats | top-row ring
// [kRingDepth][n−1][nthr] floats.
template <int NN, int CR, bool S1>
#ifndef OAA_ENGINE_MINB
#define OAA_ENGINE_MINB 1
#endif
__global__ void __launch_bounds__(kMaxThreads, OAA_ENGINE_MINB) oaa_engine_kernel(const EngineParams p) {
  constexpr int P = 2 * NN - 1, H = NN, P2 = (P + 1) / 2, TR = NN - 1;
  constexpr int NSB = S1 ? 3 : 2;  // spectrum buffers
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int s_item;
  constexpr int TS = q_stride(NN);
  constexpr int RS = kMaxThreads;                  // ring stride (floats per ring row)
  const int BW = p.BW;
  const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31;
  constexpr int qsz = H * P * TS;                  // float2 per Q buffer
  const int CIN_S = S1 ? p.Cin : CR;               // inner channels per spectrum buffer
  const int ssz = CIN_S * P2 * H;                  // float4 per spectrum buffer
  float2* Qs = reinterpret_cast<float2*>(smem_raw);
  float4* Ss = reinterpret_cast<float4*>(Qs + 2 * qsz);
  float* band = reinterpret_cast<float*>(Ss + (S1 ? NSB : 2 * p.CIG) * ssz);
  const int bandsz = NN * BW;                      // floats per staged channel
  // S1 reads the staged rows only at item start, when the ring is empty: they share space
  float* ring = S1 ? band : band + 2 * p.CIG * bandsz;  // [min(kRingDepth, Cout)][TR][RS]
  zero_q_tail<NN>(Qs, qsz, p.T, tid, nthr);

  // stage A lane = (t2, f1)
  const int a_t = tid / H, a_f1 = tid - (tid / H) * H;
  const bool comp = tid < p.ncomp;                 // compute lane (else: publisher warp)
  const bool laneA = comp && a_t < p.T;
  const int a_qoff = a_f1 * P * TS + a_t;          // this lane's Q[f1][0][t2]
  // The release that publishes progress costs a full memory fence; a dedicated warp
  // with no stores of its own issues it, so the compute warps never wait on it.
  const int pub_tid = (nthr > p.ncomp) ? p.ncomp : 0;
  // stage B lane = output column j
  const bool laneB = comp && tid < p.Ro;
  const unsigned bmask = __ballot_sync(0xffffffffu, laneB);
  const int leader = bmask ? __ffs(bmask) - 1 : 0;
  const ColGeo cg = col_geo<NN>(tid + p.off, p.T);
  const size_t plane_sz = (size_t)p.Ro * p.Ro;

  for (;;) {
    __syncthreads();  // previous item fully done with smem / s_item
    if (tid == 0) s_item = atomicAdd(p.counter, 1);
    __syncthreads();
    const int item = s_item;
    if (item >= p.num_items) break;
    const int b = item / p.T, t1 = item - (item / p.T) * p.T;
    const bool has_pred = (t1 > 0) && (TR > 0);
    const int* pred_flag = p.flags + item - 1;
    const float* in_b = p.in + (size_t)b * p.Cin * p.R * p.R;
    const int I0 = t1 * NN - p.off;  // output row of block row p1 = 0
    int seen = 0, inflight = 0;      // predecessor progress (see wait_flag)
    // rows of this tile row inside the output window, as a bit mask over p1
    unsigned rows = 0;
#pragma unroll
    for (int p1 = 0; p1 < P; ++p1)
      if (I0 + p1 >= 0 && I0 + p1 < p.Ro) rows |= 1u << p1;
    // column pointer of block row 0 in output channel 0 (may point outside; only
    // dereferenced for rows in `rows`)
    float* colp = p.out + (size_t)b * p.Cout * plane_sz + (ptrdiff_t)I0 * p.Ro + tid;

    // finish the top rows of output channel c: predecessor's partial rows + ours
    auto finalize = [&](int c, const float (&pend)[TR > 0 ? TR : 1]) {
      float* cp = colp + (size_t)c * plane_sz;
      const float* rg = ring + (c % kRingDepth) * TR * RS + tid;
#pragma unroll
      for (int p1 = 0; p1 < TR; ++p1)
        if ((rows >> p1) & 1u) __stcs(cp + (ptrdiff_t)p1 * p.Ro, pend[p1] + rg[p1 * RS]);
    };
    auto prefetch = [&](int c, float (&pend)[TR > 0 ? TR : 1]) {
      const float* cp = colp + (size_t)c * plane_sz;
#pragma unroll
      for (int p1 = 0; p1 < TR; ++p1)
        pend[p1] = ((rows >> p1) & 1u) ? __ldcg(cp + (ptrdiff_t)p1 * p.Ro) : 0.f;
    };

    // Stage B of output channel cb, split so that it can be software-pipelined against
    // stage A of the next channel:  pre_b (before the barrier-delimited block) waits for
    // the predecessor and prefetches the partial rows channel cb − kRingDepth will be
    // added onto; do_b stores this tile row's rows of channel cb, parks its top rows in
    // the ring and finalises channel cb − kRingDepth.
    const unsigned rowsB = laneB ? rows : 0u;
    auto pre_b = [&](int cb, float (&pend)[TR > 0 ? TR : 1]) -> bool {
      const bool fin = laneB && has_pred && cb >= kRingDepth;
      if (fin) {
        wait_flag(pred_flag, cb - kRingDepth + 1, lane, leader, bmask, seen, inflight);
        prefetch(cb - kRingDepth, pend);
      }
      return fin;
    };
    auto do_b = [&](int cb, bool fin, const float (&pend)[TR > 0 ? TR : 1]) {
      float y[P];
      stage_b_column<NN>(Qs + (cb & 1) * qsz, cg, y);
      float* cp = colp + (size_t)cb * plane_sz;
#pragma unroll
      for (int p1 = TR; p1 < P; ++p1) {
        if ((rowsB >> p1) & 1u) {
          if (p1 >= NN) __stcg(cp + (ptrdiff_t)p1 * p.Ro, y[p1]);   // partial: the next tile row adds
          else __stcs(cp + (ptrdiff_t)p1 * p.Ro, y[p1]);           // final
        }
      }
      // The partial rows of channels < cb+1 are published at the next barrier when
      // cb+1 is a publication point: every thread that stored them fences first
      // (bar.sync alone does not make other warps' global stores visible device-wide).
      if (((cb + 1) % kPublishEvery) == 0 && rowsB) fence_release();
      if (!has_pred) {
#pragma unroll
        for (int p1 = 0; p1 < TR; ++p1)
          if ((rowsB >> p1) & 1u) __stcs(cp + (ptrdiff_t)p1 * p.Ro, y[p1]);
      } else {
        if (fin) finalize(cb - kRingDepth, pend);
        float* rg = ring + (cb % kRingDepth) * TR * RS + tid;
#pragma unroll
        for (int p1 = 0; p1 < TR; ++p1) rg[p1 * RS] = y[p1];
        // issue the next flag read now; it is consumed an iteration later
        if (laneB && lane == leader && seen < cb + 2 - kRingDepth + kPublishEvery)
          inflight = ld_relaxed(pred_flag);
      }
    };
    // barrier; afterwards channels [0, done) have their bottom rows stored by everyone
    auto sync_publish = [&](int done) {
      cp_async_wait_1();  // all but the newest group (the spectrum prefetch two channels ahead)
      __syncthreads();
      if (tid == pub_tid && done > 0 && (done % kPublishEvery) == 0) st_release(p.flags + item, done);
    };
    // unpipelined channel (S2): stage A, barrier, stage B
    auto out_channel = [&](int co, const float (&yr)[P], const float (&yi)[P]) {
      float pend[TR > 0 ? TR : 1];
      const bool fin = pre_b(co, pend);
      if (laneA) stage_a_store<NN>(yr, yi, Qs + (co & 1) * qsz + a_qoff);
      sync_publish(co);
      if (laneB) do_b(co, fin, pend);
    };

    if constexpr (S1) {
      // stage the item's input rows and the first two output channels' spectra
      for (int c = 0; c < p.Cin; ++c)
        stage_rows(band + c * bandsz, BW, in_b + (size_t)c * p.R * p.R, p.R, t1 * NN, NN, 0, BW, tid, nthr);
      for (int co = 0; co < 2 && co < p.Cout; ++co)
        for (int e = tid; e < ssz; e += nthr) cp_async16(Ss + co * ssz + e, p.spec + (size_t)co * ssz + e);
      cp_async_commit();
      cp_async_wait_all();
      __syncthreads();
      float xr[CR][P], xi[CR][P];
#pragma unroll
      for (int c = 0; c < CR; ++c)
#pragma unroll
        for (int f2 = 0; f2 < P; ++f2) { xr[c][f2] = 0.f; xi[c][f2] = 0.f; }
      if (laneA) {
        float cf[NN], sf[NN];  // this lane's column twiddles e^{−iθ f1 p1}
#pragma unroll
        for (int p1 = 0; p1 < NN; ++p1) {
          float s, c;
          sincospif(2.0f * (float)((a_f1 * p1) % P) / (float)P, &s, &c);
          cf[p1] = c;
          sf[p1] = s;
        }
#pragma unroll
        for (int c = 0; c < CR; ++c) {
          if (c < p.Cin) {
            float z[NN][NN];
            read_block<NN>(band + c * bandsz, BW, a_t * NN, z);
            block_row_spectrum<NN>(z, cf, sf, xr[c], xi[c]);
          }
        }
      }
      __syncthreads();  // staged rows consumed: the ring may now overwrite them
      // stage A of channel co for this lane (every lane runs it: lanes past the last
      // tile write unused Q columns), plus the spectrum prefetch two channels ahead
      auto stage_a = [&](int co) {
        float yr[P], yi[P];
        const float4* S = Ss + (co % NSB) * ssz + a_f1;
#pragma unroll
        for (int c = 0; c < CR; ++c) {
          if (c < p.Cin) {
#pragma unroll
            for (int q = 0; q < P2; ++q) {
              const float4 w = S[(c * P2 + q) * H];
              const int f = 2 * q;
              if (c == 0) {
                yr[f] = w.x * xr[c][f];
                yi[f] = w.x * xi[c][f];
              } else {
                yr[f] = fmaf(w.x, xr[c][f], yr[f]);
                yi[f] = fmaf(w.x, xi[c][f], yi[f]);
              }
              yr[f] = fmaf(-w.y, xi[c][f], yr[f]);
              yi[f] = fmaf(w.y, xr[c][f], yi[f]);
              if (f + 1 < P) {
                if (c == 0) {
                  yr[f + 1] = w.z * xr[c][f + 1];
                  yi[f + 1] = w.z * xi[c][f + 1];
                } else {
                  yr[f + 1] = fmaf(w.z, xr[c][f + 1], yr[f + 1]);
                  yi[f + 1] = fmaf(w.z, xi[c][f + 1], yi[f + 1]);
                }
                yr[f + 1] = fmaf(-w.w, xi[c][f + 1], yr[f + 1]);
                yi[f + 1] = fmaf(w.w, xr[c][f + 1], yi[f + 1]);
              }
            }
          }
        }
        stage_a_store<NN>(yr, yi, Qs + (co & 1) * qsz + a_qoff);
      };
      // spectrum prefetch two channels ahead (all threads, publisher warp included)
      auto prefetch_spec = [&](int co) {
        if (co + 2 < p.Cout)
          for (int e = tid; e < ssz; e += nthr)
            cp_async16(Ss + ((co + 2) % NSB) * ssz + e, p.spec + (size_t)(co + 2) * ssz + e);
        cp_async_commit();  // always (possibly empty) so wait_group 1 keeps its meaning
      };
      // software pipeline: stage A of channel it overlaps stage B of channel it−1
      if (comp) stage_a(0);
      prefetch_spec(0);
      sync_publish(0);
      for (int it = 1; it < p.Cout; ++it) {
        if (comp) {
          float pend[TR > 0 ? TR : 1];
          const bool fin = pre_b(it - 1, pend);
          stage_a(it);
          do_b(it - 1, fin, pend);
        }
        prefetch_spec(it);
        sync_publish(it);
      }
      if (comp) {
        float pend[TR > 0 ? TR : 1];
        const bool fin = pre_b(p.Cout - 1, pend);
        do_b(p.Cout - 1, fin, pend);
      }
    } else {
      float cf[NN], sf[NN];  // this lane's column twiddles e^{−iθ f1 p1}
#pragma unroll
      for (int p1 = 0; p1 < NN; ++p1) {
        float s, c;
        sincospif(2.0f * (float)((a_f1 * p1) % P) / (float)P, &s, &c);
        cf[p1] = c;
        sf[p1] = s;
      }
      // Input channels are staged CIG at a time (one barrier per group), double buffered:
      // band[2][CIG][n][BW], spectra[2][CIG][CR][P2][H].
      const int CIG = p.CIG;
      const int ngrp = (p.Cin + CIG - 1) / CIG;
      for (int c0 = 0; c0 < p.Cout; c0 += CR) {
        const int nc = min(CR, p.Cout - c0);
        const int ssz_c = nc * P2 * H;  // float4 of one input channel's chunk spectra
        float ar[CR][P], ai[CR][P];
#pragma unroll
        for (int cc = 0; cc < CR; ++cc)
#pragma unroll
          for (int f2 = 0; f2 < P; ++f2) { ar[cc][f2] = 0.f; ai[cc][f2] = 0.f; }
        auto stage_group = [&](int g) {
          const int slot = g & 1;
          for (int j = 0; j < CIG; ++j) {
            const int ci = g * CIG + j;
            if (ci >= p.Cin) break;
            stage_rows(band + (slot * CIG + j) * bandsz, BW, in_b + (size_t)ci * p.R * p.R, p.R, t1 * NN, NN, 0,
                       BW, tid, nthr);
            for (int e = tid; e < ssz_c; e += nthr)
              cp_async16(Ss + (slot * CIG + j) * ssz + e, p.spec + ((size_t)ci * p.Cout + c0) * P2 * H + e);
          }
          cp_async_commit();
        };
        stage_group(0);
        for (int g = 0; g < ngrp; ++g) {
          cp_async_wait_all();
          __syncthreads();
          if (g + 1 < ngrp) stage_group(g + 1);  // overlaps this group's compute
          if (laneA) {
            const int nci = min(CIG, p.Cin - g * CIG);
            // accumulate one input channel's row spectrum into the output accumulators
            auto accum = [&](int slot, const float (&gr)[P], const float (&gi)[P]) {
              const float4* S = Ss + slot * ssz + a_f1;
#pragma unroll
              for (int cc = 0; cc < CR; ++cc) {
                if (cc < nc) {
#pragma unroll
                  for (int q = 0; q < P2; ++q) {
                    const float4 w = S[(cc * P2 + q) * H];
                    const int f = 2 * q;
                    ar[cc][f] = fmaf(w.x, gr[f], ar[cc][f]);
                    ar[cc][f] = fmaf(-w.y, gi[f], ar[cc][f]);
                    ai[cc][f] = fmaf(w.x, gi[f], ai[cc][f]);
                    ai[cc][f] = fmaf(w.y, gr[f], ai[cc][f]);
                    if (f + 1 < P) {
                      ar[cc][f + 1] = fmaf(w.z, gr[f + 1], ar[cc][f + 1]);
                      ar[cc][f + 1] = fmaf(-w.w, gi[f + 1], ar[cc][f + 1]);
                      ai[cc][f + 1] = fmaf(w.z, gi[f + 1], ai[cc][f + 1]);
                      ai[cc][f + 1] = fmaf(w.w, gr[f + 1], ai[cc][f + 1]);
                    }
                  }
                }
              }
            };
            int j = 0;
            for (; j + 1 < nci; j += 2) {  // two independent block transforms per step (ILP)
              const int s0 = (g & 1) * CIG + j;
              float g0r[P], g0i[P], g1r[P], g1i[P];
              block_row_spectrum_smem<NN>(band + s0 * bandsz, BW, a_t * NN, cf, sf, g0r, g0i);
              block_row_spectrum_smem<NN>(band + (s0 + 1) * bandsz, BW, a_t * NN, cf, sf, g1r, g1i);
              accum(s0, g0r, g0i);
              accum(s0 + 1, g1r, g1i);
            }
            if (j < nci) {
              const int s0 = (g & 1) * CIG + j;
              float gr[P], gi[P];
              block_row_spectrum_smem<NN>(band + s0 * bandsz, BW, a_t * NN, cf, sf, gr, gi);
              accum(s0, gr, gi);
            }
          }
        }
        __syncthreads();  // all lanes done with band / spectra before the next chunk
        cp_async_commit();  // empty group: keeps wait_group 1 in out_channel exact
#pragma unroll
        for (int cc = 0; cc < CR; ++cc)
          if (cc < nc) out_channel(c0 + cc, ar[cc], ai[cc]);
      }
    }

    // item end: publish everything, then finish the deferred channels
    if (laneB) fence_release();
    cp_async_wait_all();
    __syncthreads();
    if (tid == pub_tid) st_release(p.flags + item, p.Cout);
    if (laneB && has_pred) {
      wait_flag(pred_flag, p.Cout, lane, leader, bmask, seen, inflight);
      for (int c = max(0, p.Cout - kRingDepth); c < p.Cout; ++c) {
        float pend[TR > 0 ? TR : 1];
        prefetch(c, pend);
        finalize(c, pend);
      }
    }
  }
}

// ------------------------------------------------------------------ TMEM helpers
// Each thread owns one TMEM lane (32·(warp % 4) + lane) and reads / writes consecutive
// 32-bit columns of it (shape 32x32b).  All tcgen05 ops are warp-collective.
__device__ __forceinline__ void tmem_ld16(uint32_t ta, float* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]),
        "=f"(v[8]), "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]), "=f"(v[14]), "=f"(v[15])
      : "r"(ta));
}
__device__ __forceinline__ void tmem_st16(uint32_t ta, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(ta),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
      "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]));
}
__device__ __forceinline__ void tmem_ld8(uint32_t ta, float* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
               : "r"(ta));
}
__device__ __forceinline__ void tmem_st8(uint32_t ta, const float* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta), "f"(v[0]),
               "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]));
}
// 32 consecutive 32-bit TMEM columns of this thread's lane
__device__ __forceinline__ void tm_ld32(uint32_t ta, float* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]),
        "=f"(v[8]), "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]), "=f"(v[14]), "=f"(v[15]),
        "=f"(v[16]), "=f"(v[17]), "=f"(v[18]), "=f"(v[19]), "=f"(v[20]), "=f"(v[21]), "=f"(v[22]), "=f"(v[23]),
        "=f"(v[24]), "=f"(v[25]), "=f"(v[26]), "=f"(v[27]), "=f"(v[28]), "=f"(v[29]), "=f"(v[30]), "=f"(v[31])
      : "r"(ta));
}
__device__ __forceinline__ void tm_st32(uint32_t ta, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(ta),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
      "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]), "f"(v[16]), "f"(v[17]), "f"(v[18]),
      "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]), "f"(v[24]), "f"(v[25]), "f"(v[26]), "f"(v[27]),
      "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31]));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// TMEM columns per thread of the S1 engine: the input row spectra (CR channels, 2P
// floats each, in whole 16-column loads) + the deferred top rows (kTRing channels × 8).
constexpr int kTRing = 4;     // deferred channels per lane (TMEM ring)
constexpr int kTPublish = 2;  // progress published every kTPublish channels, one channel late
static_assert(kTRing >= kTPublish + 2, "ring must cover the publication lag");
__host__ __device__ constexpr int s1t_xcols(int n) { return ((2 * (2 * n - 1) + 15) / 16) * 16; }
__host__ __device__ constexpr int s1t_cols_per_thread(int n, int cr) { return cr * s1t_xcols(n) + kTRing * 8; }
// columns allocated per CTA: two warps share every TMEM lane (8 warps / 4 quadrants)
__host__ __device__ constexpr int s1t_alloc_cols(int n, int cr) {
  return (2 * s1t_cols_per_thread(n, cr) <= 32) ? 32 : (2 * s1t_cols_per_thread(n, cr) <= 64) ? 64
       : (2 * s1t_cols_per_thread(n, cr) <= 128) ? 128 : (2 * s1t_cols_per_thread(n, cr) <= 256) ? 256 : 512;
}

// ------------------------------------------------------------------ S1 engine, TMEM
// Input-stationary engine (forward at small C) with the per-lane input row spectra and
// the deferred overlap rows held in tensor memory instead of registers, so two CTAs
// (16 warps) fit on an SM.  Same algorithm and protocol as oaa_engine_kernel<.., S1>.
// Shared memory: Q[2][H][P][TS] float2 | spectra[3][Cin][P2][H] float4 | staged rows.
//
// LY = true: the "load-Ŷ" variant used after the tensor-core contraction (oaa_tc.cuh):
// stage A reads this lane's spectrum row of Ŷ for output channel co from D instead of
// contracting register / TMEM spectra; everything after (row IDFT, stage B, overlap-add
// protocol) is shared.  TMEM then only holds the ring.
template <int NN, int CR, bool LY>
__global__ void __launch_bounds__(kMaxThreads, 2) oaa_engine_s1t_kernel(const EngineParams p) {
  constexpr int P = 2 * NN - 1, H = NN, P2 = (P + 1) / 2, TR = NN - 1;
  constexpr int NSB = 3;
  constexpr int TS = q_stride(NN);
  constexpr int XC = s1t_xcols(NN);                 // TMEM columns per channel
  constexpr int NX16 = XC / 16;
  constexpr int RING0 = LY ? 0 : CR * XC;           // first ring column
  constexpr int ACOLS = s1t_alloc_cols(NN, LY ? 0 : CR);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int s_item;
  __shared__ uint32_t s_tmem;
  const int BW = p.BW;
  const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31, warp = tid >> 5;
  constexpr int qsz = H * P * TS;
  const int ssz = p.Cin * P2 * H;
  float2* Qs = reinterpret_cast<float2*>(smem_raw);
  float4* Ss = reinterpret_cast<float4*>(Qs + 2 * qsz);
  float* band = reinterpret_cast<float*>(Ss + NSB * ssz);
  const int bandsz = NN * BW;
  zero_q_tail<NN>(Qs, qsz, p.T, tid, nthr);

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&s_tmem)),
                 "n"(ACOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tbase = s_tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) & 1) * (ACOLS / 2);

  const int a_t = tid / H, a_f1 = tid - (tid / H) * H;
  const bool comp = tid < p.ncomp;
  const bool laneA = comp && a_t < p.T;
  const int a_qoff = a_f1 * P * TS + a_t;
  const int pub_tid = (nthr > p.ncomp) ? p.ncomp : 0;
  const bool laneB = comp && tid < p.Ro;
  const unsigned bmask = __ballot_sync(0xffffffffu, laneB);
  const int leader = bmask ? __ffs(bmask) - 1 : 0;
  const ColGeo cg = col_geo<NN>(tid + p.off, p.T);
  const size_t plane_sz = (size_t)p.Ro * p.Ro;

  for (;;) {
    __syncthreads();
    if (tid == 0) s_item = atomicAdd(p.counter, 1);
    __syncthreads();
    const int item = s_item;
    if (item >= p.num_items) break;
    const int bl = item / p.T, t1 = item - (item / p.T) * p.T;
    const int b = bl + (LY ? p.b0 : 0);
    const bool has_pred = (t1 > 0) && (TR > 0);
    const int* pred_flag = p.flags + item - 1;
    const float* in_b = LY ? nullptr : p.in + (size_t)b * p.Cin * p.R * p.R;
    const int I0 = t1 * NN - p.off;
    int seen = 0, inflight = 0;
    unsigned rows = 0;
#pragma unroll
    for (int p1 = 0; p1 < P; ++p1)
      if (I0 + p1 >= 0 && I0 + p1 < p.Ro) rows |= 1u << p1;
    const unsigned rowsB = laneB ? rows : 0u;
    float* colp = p.out + (size_t)b * p.Cout * plane_sz + (ptrdiff_t)I0 * p.Ro + tid;

    // stage input rows + the first two spectra
    if (!LY) {
      for (int c = 0; c < p.Cin; ++c)
        stage_rows(band + c * bandsz, BW, in_b + (size_t)c * p.R * p.R, p.R, t1 * NN, NN, 0, BW, tid, nthr);
      for (int co = 0; co < 2 && co < p.Cout; ++co)
        for (int e = tid; e < ssz; e += nthr) cp_async16(Ss + co * ssz + e, p.spec + (size_t)co * ssz + e);
    }
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();
    // this lane's input row spectra → TMEM (lanes past the last tile store zeros)
    if (!LY) {
      float cf[NN], sf[NN];
#pragma unroll
      for (int p1 = 0; p1 < NN; ++p1) {
        float s, c;
        sincospif(2.0f * (float)((a_f1 * p1) % P) / (float)P, &s, &c);
        cf[p1] = c;
        sf[p1] = s;
      }
#pragma unroll
      for (int c = 0; c < CR; ++c) {
        float xb[XC];
#pragma unroll
        for (int q = 0; q < XC; ++q) xb[q] = 0.f;
        if (laneA && c < p.Cin) {
          float z[NN][NN], xr[P], xi[P];
          read_block<NN>(band + c * bandsz, BW, a_t * NN, z);
          block_row_spectrum<NN>(z, cf, sf, xr, xi);
#pragma unroll
          for (int f = 0; f < P; ++f) { xb[f] = xr[f]; xb[P + f] = xi[f]; }
        }
#pragma unroll
        for (int q = 0; q < NX16; ++q) tmem_st16(tbase + c * XC + 16 * q, xb + 16 * q);
      }
      tmem_wait_st();
    }

    constexpr unsigned kAll = (1u << P) - 1u;
    const bool fullB = rowsB == kAll;  // interior tile row: no per-row bounds checks
    const ptrdiff_t Ro = p.Ro;
    auto prefetch = [&](int c, float (&pend)[TR > 0 ? TR : 1]) {
      const float* cp = colp + (size_t)c * plane_sz;
      if (fullB) {
#pragma unroll
        for (int p1 = 0; p1 < TR; ++p1) { pend[p1] = __ldcg(cp); cp += Ro; }
      } else {
#pragma unroll
        for (int p1 = 0; p1 < TR; ++p1)
          pend[p1] = ((rowsB >> p1) & 1u) ? __ldcg(cp + (ptrdiff_t)p1 * Ro) : 0.f;
      }
    };
    auto store_rows = [&](float* cp, const float* v, int p_lo, int p_hi, bool partial_from_n) {
      if (fullB) {
        float* r = cp + (ptrdiff_t)p_lo * Ro;
#pragma unroll
        for (int p1 = 0; p1 < P; ++p1) {
          if (p1 >= p_lo && p1 < p_hi) {
            if (partial_from_n && p1 >= NN) __stcg(r, v[p1]);
            else __stcs(r, v[p1]);
            r += Ro;
          }
        }
      } else {
#pragma unroll
        for (int p1 = 0; p1 < P; ++p1)
          if (p1 >= p_lo && p1 < p_hi && ((rowsB >> p1) & 1u)) {
            if (partial_from_n && p1 >= NN) __stcg(cp + (ptrdiff_t)p1 * Ro, v[p1]);
            else __stcs(cp + (ptrdiff_t)p1 * Ro, v[p1]);
          }
      }
    };
    auto pre_b = [&](int cb, float (&pend)[TR > 0 ? TR : 1]) -> bool {
      const bool fin = laneB && has_pred && cb >= kTRing;
      if (fin) {
        wait_flag(pred_flag, cb - kTRing + 1, lane, leader, bmask, seen, inflight);  // publication lags ≤ kTPublish+1
        prefetch(cb - kTRing, pend);
      }
      return fin;
    };
    // stage B of channel cb (warp-uniform: TMEM ring accesses are collective)
    auto do_b = [&](int cb, bool fin, const float (&pend)[TR > 0 ? TR : 1]) {
      float y[P];
      stage_b_column<NN>(Qs + (cb & 1) * qsz, cg, y);
      float* cp = colp + (size_t)cb * plane_sz;
      // Channels < cb are published at the barrier that follows when cb is a
      // publication point.  Every thread that stored their partial rows fences first;
      // the fence sits BEFORE this channel's stores, so the stores it waits for were
      // issued an iteration ago and have normally landed (a cheap fence).
      if ((cb % kTPublish) == 0 && cb > 0 && rowsB) fence_release();
      store_rows(cp, y, TR, P, true);
      if (!has_pred) {
        store_rows(cp, y, 0, TR, false);
      } else if (TR > 0) {
        const uint32_t slot = tbase + RING0 + (cb % kTRing) * 8;
        float old[8];
        __syncwarp();
        tmem_ld8(slot, old);  // channel cb − kTRing's top rows (same slot)
        tmem_wait_ld();
        if (fin) {
          float sum[P];
#pragma unroll
          for (int p1 = 0; p1 < P; ++p1) sum[p1] = (p1 < TR) ? pend[p1] + old[p1] : 0.f;
          store_rows(colp + (size_t)(cb - kTRing) * plane_sz, sum, 0, TR, false);
        }
        float nw[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) nw[q] = (q < TR) ? y[q] : 0.f;
        tmem_st8(slot, nw);
        if (laneB && lane == leader && seen < cb + 2 - kTRing + kTPublish) inflight = ld_relaxed(pred_flag);
      }
    };
    // barrier after stage B of channel cb: channels [0, cb) are fenced by everyone
    auto sync_publish = [&](int cb) {
      cp_async_wait_1();
      tmem_wait_st();
      __syncthreads();
      if (tid == pub_tid && cb > 0 && (cb % kTPublish) == 0) st_release(p.flags + item, cb);
    };
    // LY: this lane's Ŷ row for output channel co (bins f = f1·P + f2, zero past the tiles)
    // LY: this lane's Ŷ row (bins f1·P + f2) of the next output channel, loaded one
    // channel ahead into registers so the loads fly during the previous channel's work
    const float* dlane = LY ? p.D + (size_t)(a_f1 * P) * 2 * p.Cout * p.BTc + (size_t)(bl * p.T + t1) * p.T + a_t
                            : nullptr;
    float yrn[LY ? P : 1], yin[LY ? P : 1];
    auto load_y = [&](int co) {
      if constexpr (LY) {
#pragma unroll
        for (int f2 = 0; f2 < P; ++f2) {
          const float* d = dlane + ((size_t)f2 * 2 * p.Cout + co) * p.BTc;
          yrn[f2] = laneA ? __ldg(d) : 0.f;
          yin[f2] = laneA ? __ldg(d + (size_t)p.Cout * p.BTc) : 0.f;
        }
      }
    };
    auto stage_a = [&](int co) {
      float yr[P], yi[P];
      if constexpr (LY) {
#pragma unroll
        for (int f2 = 0; f2 < P; ++f2) { yr[f2] = yrn[f2]; yi[f2] = yin[f2]; }
        if (co + 1 < p.Cout) load_y(co + 1);
        stage_a_store<NN>(yr, yi, Qs + (co & 1) * qsz + a_qoff);
        return;
      }
      const float4* S = Ss + (co % NSB) * ssz + a_f1;
      __syncwarp();  // tcgen05.ld is warp-collective: reconverge after divergent code
#pragma unroll
      for (int c = 0; c < CR; ++c) {
        if (c < p.Cin) {
          float xb[XC];
#pragma unroll
          for (int q = 0; q < NX16; ++q) tmem_ld16(tbase + c * XC + 16 * q, xb + 16 * q);
          tmem_wait_ld();
#pragma unroll
          for (int q = 0; q < P2; ++q) {
            const float4 w = S[(c * P2 + q) * H];
            const int f = 2 * q;
            const float x0r = xb[f], x0i = xb[P + f];
            if (c == 0) { yr[f] = w.x * x0r; yi[f] = w.x * x0i; }
            else { yr[f] = fmaf(w.x, x0r, yr[f]); yi[f] = fmaf(w.x, x0i, yi[f]); }
            yr[f] = fmaf(-w.y, x0i, yr[f]);
            yi[f] = fmaf(w.y, x0r, yi[f]);
            if (f + 1 < P) {
              const float x1r = xb[f + 1], x1i = xb[P + f + 1];
              if (c == 0) { yr[f + 1] = w.z * x1r; yi[f + 1] = w.z * x1i; }
              else { yr[f + 1] = fmaf(w.z, x1r, yr[f + 1]); yi[f + 1] = fmaf(w.z, x1i, yi[f + 1]); }
              yr[f + 1] = fmaf(-w.w, x1i, yr[f + 1]);
              yi[f + 1] = fmaf(w.w, x1r, yi[f + 1]);
            }
          }
        }
      }
      stage_a_store<NN>(yr, yi, Qs + (co & 1) * qsz + a_qoff);
    };
    auto prefetch_spec = [&](int co) {
      if (!LY && co + 2 < p.Cout)
        for (int e = tid; e < ssz; e += nthr)
          cp_async16(Ss + ((co + 2) % NSB) * ssz + e, p.spec + (size_t)(co + 2) * ssz + e);
      cp_async_commit();
    };

    if (LY && comp) load_y(0);
    if (comp) stage_a(0);
    prefetch_spec(0);
    sync_publish(0);
    for (int it = 1; it < p.Cout; ++it) {
      if (comp) {
        float pend[TR > 0 ? TR : 1];
        const bool fin = pre_b(it - 1, pend);
        stage_a(it);
        do_b(it - 1, fin, pend);
      }
      prefetch_spec(it);
      sync_publish(it - 1);
    }
    if (comp) {
      float pend[TR > 0 ? TR : 1];
      const bool fin = pre_b(p.Cout - 1, pend);
      do_b(p.Cout - 1, fin, pend);
    }
    // item end: fence + publish, then finish the deferred channels
    if (laneB) fence_release();
    cp_async_wait_all();
    tmem_wait_st();
    __syncthreads();
    if (tid == pub_tid) st_release(p.flags + item, p.Cout);
    if (comp && has_pred && TR > 0) {
      if (laneB) wait_flag(pred_flag, p.Cout, lane, leader, bmask, seen, inflight);
      for (int c = max(0, p.Cout - kTRing); c < p.Cout; ++c) {
        float pend[TR > 0 ? TR : 1];
        prefetch(c, pend);
        float old[8];
        __syncwarp();
        tmem_ld8(tbase + RING0 + (c % kTRing) * 8, old);
        tmem_wait_ld();
        float sum[P];
#pragma unroll
        for (int p1 = 0; p1 < P; ++p1) sum[p1] = (p1 < TR) ? pend[p1] + old[p1] : 0.f;
        store_rows(colp + (size_t)c * plane_sz, sum, 0, TR, false);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_tmem), "n"(ACOLS));
}

// ------------------------------------------------------------------ bwd_filter
// Stage rows r0..r0+NROWS of `nplanes` consecutive R×R planes (plane stride R·R),
// columns [c0, c0+ncols), into dst[plane][row][ld] (zero outside).  Warps own rows,
// lanes own columns, and the plane loop only bumps pointers, so a copy costs a handful
// of instructions (the rows are not 16-byte aligned in general: M = N−n+1 is odd).
template <int NROWS>
__device__ __forceinline__ void stage_planes_rows(float* dst, int ld, const float* __restrict__ base,
                                                  int nplanes, int R, int r0, int c0, int ncols, int tid,
                                                  int nthr) {
  const int lane = tid & 31, warp = tid >> 5, nwarps = nthr >> 5;
  const size_t pstride = (size_t)R * R;
  for (int rr = warp; rr < NROWS; rr += nwarps) {
    const int r = r0 + rr;
    const bool rok = r >= 0 && r < R;
    for (int cc = lane; cc < ncols; cc += 32) {
      const int q = c0 + cc;
      const bool ok = rok && q >= 0 && q < R;
      const float* src = ok ? base + (size_t)r * R + q : base;
      float* d = dst + rr * ld + cc;
      for (int pl = 0; pl < nplanes; ++pl) {
        cp_async4(d, src, ok);
        if (ok) src += pstride;
        d += NROWS * ld;
      }
    }
  }
}

// Shared memory: x window rows [CR][P][XW] floats | Ξ̂ for the item's tiles [Td][CR][P][H]
// float2 | dy blocks of TCH tiles [2][KG][NN][DW] floats (double buffered) | twiddles.
template <int NN, int CR>
__global__ void __launch_bounds__(kMaxThreads, 1) oaa_bwd_filter_kernel(const FilterParams p) {
  constexpr int P = 2 * NN - 1, H = NN;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int kk = tid / H, f1 = tid - (tid / H) * H;
  const int k0 = blockIdx.y * p.KG;
  const int k = k0 + kk;
  const int nk = min(p.KG, p.K - k0);
  const bool laneK = kk < nk;
  const int XW = p.XW, DW = p.DW;
  const int dysz = p.KG * NN * DW;
  float* xwin = reinterpret_cast<float*>(smem_raw);                        // [CR][P][XW]
  float2* xs = reinterpret_cast<float2*>(xwin + CR * P * XW);              // [Td][CR][P][H]
  float* dyb = reinterpret_cast<float*>(xs + (size_t)p.Td * CR * P * H);   // [2][KG][NN][DW]
  float2* tw = reinterpret_cast<float2*>(dyb + 2 * dysz);                  // [P] (cos, sin)(2πm/P)
  if (tid < P) {
    float s, c;
    sincospif(2.0f * (float)tid / (float)P, &s, &c);
    tw[tid] = make_float2(c, s);
  }
  float cf[NN], sf[NN];
#pragma unroll
  for (int p1 = 0; p1 < NN; ++p1) {
    float s, c;
    sincospif(2.0f * (float)((f1 * p1) % P) / (float)P, &s, &c);
    cf[p1] = c;
    sf[p1] = s;
  }
  const int items = p.B * p.Td;
  const int w0 = p.off - (NN - 1);  // x-window origin relative to the dy block origin
  const int nchunks = (p.Td + p.TCH - 1) / p.TCH;
  for (int c0 = 0; c0 < p.C; c0 += CR) {
    const int nc = min(CR, p.C - c0);
    float ar[CR][P], ai[CR][P];
#pragma unroll
    for (int cc = 0; cc < CR; ++cc)
#pragma unroll
      for (int f2 = 0; f2 < P; ++f2) { ar[cc][f2] = 0.f; ai[cc][f2] = 0.f; }
    for (int item = blockIdx.x; item < items; item += p.G) {
      const int b = item / p.Td, t1 = item - (item / p.Td) * p.Td;
      const float* dyk = p.dy + ((size_t)b * p.K + k0) * p.M * p.M;
      __syncthreads();  // previous item done with xwin / xs / dyb
      // x rows of this item's windows (zero outside x) and the first dy chunk
      stage_planes_rows<P>(xwin, XW, p.x + ((size_t)b * p.C + c0) * p.N * p.N, nc, p.N, t1 * NN + w0, w0, XW,
                           tid, nthr);
      stage_planes_rows<NN>(dyb, DW, dyk, nk, p.M, t1 * NN, 0, min(p.TCH, p.Td) * NN, tid, nthr);
      cp_async_commit();
      cp_async_wait_all();
      __syncthreads();
      // Ξ̂ of every window of the item: tasks (tile t2, channel cc, row fr)
      const int ntask = p.Td * nc * H;
      for (int task = tid; task < ntask; task += nthr) {
        const int fr = task % H;
        const int cc = (task / H) % nc;
        const int t2 = task / (H * nc);
        const float* src = xwin + cc * P * XW + t2 * NN;
        float tc[P], ts[P];
#pragma unroll
        for (int p1 = 0; p1 < P; ++p1) {
          const float2 t = tw[(fr * p1) % P];
          tc[p1] = t.x;
          ts[p1] = t.y;
        }
        float rr[P], ri[P];
#pragma unroll
        for (int p2 = 0; p2 < P; ++p2) {
          float a = src[p2], bb = 0.f;
#pragma unroll
          for (int p1 = 1; p1 < P; ++p1) {
            const float v = src[p1 * XW + p2];
            a = fmaf(v, tc[p1], a);
            bb = fmaf(-v, ts[p1], bb);
          }
          rr[p2] = a;
          ri[p2] = bb;
        }
        float xr[P], xi[P];
        dft<P, -1>(rr, ri, xr, xi);
        float2* dst = xs + ((size_t)(t2 * CR + cc) * P) * H + fr;
#pragma unroll
        for (int f2 = 0; f2 < P; ++f2) dst[f2 * H] = make_float2(xr[f2], xi[f2]);
      }
      // dy blocks, TCH tiles per chunk, the next chunk staged while this one computes
      for (int ch = 0; ch < nchunks; ++ch) {
        const int tc0 = ch * p.TCH;
        const int ntc = min(p.TCH, p.Td - tc0);
        cp_async_wait_all();
        __syncthreads();  // chunk ch landed, Ξ̂ written, chunk ch−1's buffer free
        if (ch + 1 < nchunks) {
          const int t0n = tc0 + p.TCH;
          stage_planes_rows<NN>(dyb + ((ch + 1) & 1) * dysz, DW, dyk, nk, p.M, t1 * NN, t0n * NN,
                                min(p.TCH, p.Td - t0n) * NN, tid, nthr);
          cp_async_commit();
        }
        if (laneK) {
          const float* db = dyb + (ch & 1) * dysz + kk * NN * DW;
          // accumulate conj(Ĝ)·Ξ̂ of one block into the lane's dŴ row
          auto accum = [&](int tt, const float (&gr)[P], const float (&gi)[P]) {
            const float2* src = xs + ((size_t)((tc0 + tt) * CR) * P) * H + f1;
#pragma unroll
            for (int cc = 0; cc < CR; ++cc) {
              if (cc < nc) {
#pragma unroll
                for (int f2 = 0; f2 < P; ++f2) {
                  const float2 X = src[(cc * P + f2) * H];
                  ar[cc][f2] = fmaf(gr[f2], X.x, ar[cc][f2]);
                  ar[cc][f2] = fmaf(gi[f2], X.y, ar[cc][f2]);
                  ai[cc][f2] = fmaf(gr[f2], X.y, ai[cc][f2]);
                  ai[cc][f2] = fmaf(-gi[f2], X.x, ai[cc][f2]);
                }
              }
            }
          };
          int tt = 0;
          for (; tt + 1 < ntc; tt += 2) {  // two independent block transforms per step (ILP)
            float g0r[P], g0i[P], g1r[P], g1i[P];
            block_row_spectrum_smem<NN>(db, DW, tt * NN, cf, sf, g0r, g0i);
            block_row_spectrum_smem<NN>(db, DW, (tt + 1) * NN, cf, sf, g1r, g1i);
            accum(tt, g0r, g0i);
            accum(tt + 1, g1r, g1i);
          }
          if (tt < ntc) {
            float gr[P], gi[P];
            block_row_spectrum_smem<NN>(db, DW, tt * NN, cf, sf, gr, gi);
            accum(tt, gr, gi);
          }
        }
      }
    }
    if (laneK) {
#pragma unroll
      for (int cc = 0; cc < CR; ++cc) {
        if (cc < nc) {
          float2* dst =
              p.partial + ((((size_t)blockIdx.x * p.K + k) * p.C + c0 + cc) * P) * H + f1;
#pragma unroll
          for (int f2 = 0; f2 < P; ++f2) dst[f2 * H] = make_float2(ar[cc][f2], ai[cc][f2]);
        }
      }
    }
  }
}

#ifdef OAA_DEFINE_AUX_KERNELS  // defined in exactly one translation unit (oaa_abi.cu)
// partial[G][K][C][P][H] → dw[K][C][n][n].  One CTA of 512 threads per (k, c): thread
// (j, t) sums the partial spectra g ≡ j (mod 4) of bin t in fp64 (four interleaved chains,
// up to 64 loads per bin in flight), the four sums are combined in a fixed order --
// bitwise reproducible -- then the inverse DFT and lag read-out.
__global__ void __launch_bounds__(512) oaa_filter_finalize_kernel(const float2* __restrict__ partial,
                                                                  float* __restrict__ dw, int G, int K, int C,
                                                                  int n, int P) {
  const int H = (P + 1) / 2, bins = P * H;  // P = 2n − 1, or b + n − 1 for blocks b ≠ n (odd)
  const int kc = blockIdx.x;
  extern __shared__ double2 S[];  // [P][H]
  __shared__ double tc[16], ts[16];  // cos / sin (2π m / P)
  __shared__ double2 part[4][128];
  if (threadIdx.x < P) sincospi(2.0 * (double)threadIdx.x / (double)P, &ts[threadIdx.x], &tc[threadIdx.x]);
  const size_t gstride = (size_t)K * C * bins;
  {
    const int j = threadIdx.x >> 7, t = threadIdx.x & 127;
    if (t < bins) {
      const float2* src = partial + (size_t)kc * bins + t;
      double sr[4] = {0.0, 0.0, 0.0, 0.0}, si[4] = {0.0, 0.0, 0.0, 0.0};
      int g = j;
      // 16 loads in flight per thread (the sum is latency-bound, not bandwidth-bound)
      for (; g + 60 < G; g += 64) {
        float2 v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = __ldg(src + (size_t)(g + 4 * u) * gstride);
#pragma unroll
        for (int u = 0; u < 16; ++u) { sr[u & 3] += (double)v[u].x; si[u & 3] += (double)v[u].y; }
      }
      for (; g + 12 < G; g += 16) {
        float2 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = __ldg(src + (size_t)(g + 4 * u) * gstride);
#pragma unroll
        for (int u = 0; u < 4; ++u) { sr[u] += (double)v[u].x; si[u] += (double)v[u].y; }
      }
      for (int u = 0; g < G; g += 4, ++u) {
        const float2 v = __ldg(src + (size_t)g * gstride);
        sr[u] += (double)v.x;
        si[u] += (double)v.y;
      }
      part[j][t] = make_double2((sr[0] + sr[1]) + (sr[2] + sr[3]), (si[0] + si[1]) + (si[2] + si[3]));
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < bins; t += blockDim.x)
    S[t] = make_double2((part[0][t].x + part[1][t].x) + (part[2][t].x + part[3][t].x),
                        (part[0][t].y + part[1][t].y) + (part[2][t].y + part[3][t].y));
  __syncthreads();
  const double inv = 1.0 / ((double)P * (double)P);
  for (int t = threadIdx.x; t < n * n; t += blockDim.x) {
    const int u = t / n, v = t - (t / n) * n;
    const int l1 = n - 1 - u, l2 = n - 1 - v;
    double acc = 0.0;
    int m1 = 0;  // f1·l1 mod P, kept incrementally
    for (int f1 = 0; f1 < H; ++f1) {
      const double wgt = (f1 == 0) ? 1.0 : 2.0;
      double a = 0.0;
      int m = m1;  // (f1·l1 + f2·l2) mod P
      for (int f2 = 0; f2 < P; ++f2) {
        const double2 z = S[f2 * H + f1];
        a += z.x * tc[m] - z.y * ts[m];
        m += l2;
        if (m >= P) m -= P;
      }
      acc += wgt * a;
      m1 += l1;
      if (m1 >= P) m1 -= P;
    }
    dw[(size_t)kc * n * n + t] = (float)(acc * inv);
  }
}

// The same for few partial spectra (G < 32, e.g. the tensor-core weight gradient's splits):
// one warp per (k, c), 8 per CTA -- the many (k, c) pairs of a wide layer (AlexNet-like:
// 24 576) then take 3 072 CTAs instead of 24 576.  Fixed summation order (g ascending).
__global__ void __launch_bounds__(256) oaa_filter_finalize_small_kernel(const float2* __restrict__ partial,
                                                                        float* __restrict__ dw, int G, int K, int C,
                                                                        int n, int P) {
  const int H = (P + 1) / 2, bins = P * H;
  __shared__ double tc[16], ts[16];
  __shared__ double2 S[8][120];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kc = blockIdx.x * 8 + warp;
  if (threadIdx.x < P) sincospi(2.0 * (double)threadIdx.x / (double)P, &ts[threadIdx.x], &tc[threadIdx.x]);
  __syncthreads();
  if (kc >= K * C) return;
  const size_t gstride = (size_t)K * C * bins;
  for (int t = lane; t < bins; t += 32) {
    const float2* src = partial + (size_t)kc * bins + t;
    double sr = 0.0, si = 0.0;
    for (int g = 0; g < G; ++g) {
      const float2 v = __ldg(src + (size_t)g * gstride);
      sr += (double)v.x;
      si += (double)v.y;
    }
    S[warp][t] = make_double2(sr, si);
  }
  __syncwarp();
  const double inv = 1.0 / ((double)P * (double)P);
  for (int t = lane; t < n * n; t += 32) {
    const int u = t / n, v = t - (t / n) * n;
    const int l1 = n - 1 - u, l2 = n - 1 - v;
    double acc = 0.0;
    int m1 = 0;
    for (int f1 = 0; f1 < H; ++f1) {
      const double wgt = (f1 == 0) ? 1.0 : 2.0;
      double a = 0.0;
      int m = m1;
      for (int f2 = 0; f2 < P; ++f2) {
        const double2 z = S[warp][f2 * H + f1];
        a += z.x * tc[m] - z.y * ts[m];
        m += l2;
        if (m >= P) m -= P;
      }
      acc += wgt * a;
      m1 += l1;
      if (m1 >= P) m1 -= P;
    }
    dw[(size_t)kc * n * n + t] = (float)(acc * inv);
  }
}

// spec4[((a·Binner + bb)·P2 + f2/2)·H + f1].{xy|zw} = DFT_P(w_kc or flip180(w_kc))[f1][f2] / P²
// with (k, c) = loop_is_k ? (a, bb) : (bb, a); the odd last f2 slot is zero.
// One CTA per (k, c) pair (grid = K·C): the n×n kernel is staged in fp64, the row DFT
// R[p1][f2] = Σ_p2 v[p1][p2]·e^{−2πi f2 p2/P} (n terms) goes to shared memory, then each
// bin pair is Σ_p1 R[p1][f]·e^{−2πi f1 p1/P} (n terms) -- the separable 2-D DFT, fp64
// throughout, rounded to fp32 once.
// P: the transform size, 2n−1 for blocks of the kernel's size, b + n − 1 for the walker's
// larger blocks b (oaa_walk.cuh; P odd, H = P2 = (P + 1) / 2 half-spectrum rows / bin pairs).
__global__ void __launch_bounds__(128) oaa_spectrum_kernel(const float* __restrict__ w, float4* __restrict__ spec,
                                                           int K, int C, int n, int P, int flip, int loop_is_k) {
  const int H = (P + 1) / 2, P2 = (P + 1) / 2;
  __shared__ double tc[16], ts[16];  // cos / sin (2π m / P), fp64
  __shared__ double v[64];           // the kernel (flipped for bwd_data)
  __shared__ double Rr[8 * 15], Ri[8 * 15];
  const int tid = threadIdx.x;
  const int kc = blockIdx.x;  // = k·C + c
  const int k = kc / C, c = kc - (kc / C) * C;
  const float* wk = w + (size_t)kc * n * n;
  if (tid < P) sincospi(2.0 * (double)tid / (double)P, &ts[tid], &tc[tid]);
  if (tid < n * n) {
    const int p1 = tid / n, p2 = tid - (tid / n) * n;
    v[tid] = (double)(flip ? wk[(n - 1 - p1) * n + (n - 1 - p2)] : wk[tid]);
  }
  __syncthreads();
  if (tid < n * P) {
    const int p1 = tid / P, f2 = tid - (tid / P) * P;
    double sr = 0.0, si = 0.0;
    int m = 0;  // f2·p2 mod P
    for (int p2 = 0; p2 < n; ++p2) {
      const double x = v[p1 * n + p2];
      sr += x * tc[m];
      si -= x * ts[m];
      m += f2;
      if (m >= P) m -= P;
    }
    Rr[tid] = sr;
    Ri[tid] = si;
  }
  __syncthreads();
  const double inv = 1.0 / ((double)P * (double)P);
  const int a = loop_is_k ? k : c, bb = loop_is_k ? c : k, Binner = loop_is_k ? C : K;
  float4* dst = spec + (size_t)(a * Binner + bb) * P2 * H;
  for (int t = tid; t < P2 * H; t += blockDim.x) {
    const int q = t / H, f1 = t - (t / H) * H;
    const int fa = 2 * q, fb = 2 * q + 1;
    const bool hb = fb < P;
    double sra = 0.0, sia = 0.0, srb = 0.0, sib = 0.0;
    int m = 0;  // f1·p1 mod P
    for (int p1 = 0; p1 < n; ++p1) {
      const double c0 = tc[m], s0 = ts[m];
      // (R · e^{−iθ}) = (Rr c + Ri s) + i (Ri c − Rr s)
      const double ar = Rr[p1 * P + fa], ai = Ri[p1 * P + fa];
      sra += ar * c0 + ai * s0;
      sia += ai * c0 - ar * s0;
      if (hb) {
        const double br = Rr[p1 * P + fb], bi = Ri[p1 * P + fb];
        srb += br * c0 + bi * s0;
        sib += bi * c0 - br * s0;
      }
      m += f1;
      if (m >= P) m -= P;
    }
    dst[t] = make_float4((float)(sra * inv), (float)(sia * inv), hb ? (float)(srb * inv) : 0.f,
                         hb ? (float)(sib * inv) : 0.f);
  }
}
#endif  // OAA_DEFINE_AUX_KERNELS

}  // namespace oaa

namespace oaa {

// ------------------------------------------------------------------ operand producers
// Operands of the tensor-core bin GEMM (oaa_tc.cuh) are written as plain fp32 in the
// UMMA-blocked layout
//   Op[f][kc][rt][4096 floats],  kc = k/32, rt = r/128,
// each block a 128-row × 32-k tile in canonical no-swizzle K-major order.  The GEMM splits
// them for 3×TF32 in shared memory (hi = x with the low 13 mantissa bits cleared, lo = x − hi).
__device__ __forceinline__ size_t tc_idx(int f, int Kc, int RT, int r, int k) {
  return (((size_t)f * Kc + (k >> 5)) * RT + (r >> 7)) * 4096 + ((r & 127) >> 3) * 256 +
         ((k & 31) >> 2) * 32 + (r & 7) * 4 + (k & 3);
}
__device__ __forceinline__ void tc_put(float* Op, int f, int Kc, int RT, int r, int k, float v) {
  Op[tc_idx(f, Kc, RT, r, k)] = v;
}
// Pre-split variant for the small, reused A operand of fwd / bwd_data (the real-ified
// weights): Op[f][kc][h][rt][4096], h = hi | lo, so the GEMM copies both halves and its
// converter warps only split B.
__device__ __forceinline__ size_t tc_idx_split(int f, int Kc, int RT, int h, int r, int k) {
  return ((((size_t)f * Kc + (k >> 5)) * 2 + h) * RT + (r >> 7)) * 4096 + ((r & 127) >> 3) * 256 +
         ((k & 31) >> 2) * 32 + (r & 7) * 4 + (k & 3);
}
__device__ __forceinline__ void tc_put_split(float* Op, int f, int Kc, int RT, int r, int k, float v) {
  const float hi = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
  Op[tc_idx_split(f, Kc, RT, 0, r, k)] = hi;
  Op[tc_idx_split(f, Kc, RT, 1, r, k)] = v - hi;
}

// B operand: the forward spectra of every input block of a batch chunk, row
// bt = (b−b0)·T² + t1·T + t2, column c < Cin: Re X̂_c, Cinp + c: Im X̂_c (Cinp = Cin
// rounded up to 4), zero elsewhere up to 32·Kc; bin f = f1·P + f2 (half spectrum, f1 < n).
struct TileSpecParams {
  const float* in;  // [B][Cin][R][R]
  float* Xg;        // blocked [F][Kc][RTB][4096] (split: [F][Kc][hi|lo][RTB][4096])
  int Cin, R, T, b0, bc, Kc, RTB, BW, CSTR;
  int split;        // write hi / lo (for GEMMs that re-read each B tile for many M tiles)
  // fused backward (NEXT-1): the same dy-block spectra Ĝ are ALSO written as
  // the weight-gradient GEMM's A operand (oaa_filter_spectra_kernel's G mode: row k,
  // reduction j = 2·bt + {re, im}), so dy is read and transformed once for both backward
  // convolutions.  Ga == nullptr: plain tile spectra.
  float* Ga;
  int KcG, RTG;
  // overlap-and-save forward (NEXT-2), win = 1: row bt is an OUTPUT tile and its
  // spectrum is that of the (2n−1)² x-window at (t1·n + org, t2·n + org), org = o − (n−1), zero
  // outside x
  int win, org;
  int BB;  // block size (launcher: b = n, or 16 − n, R18)
};

// One CTA per (image, tile row) of the chunk.  A task is (f1, tile t2, quad of 4
// channels): its spectra go out as float4 (4 consecutive columns of one row), and the 8
// lanes of consecutive tiles of a warp fill whole 128-byte lines of the blocked layout.
// WIN (overlap-and-save): the tiles are output tiles and the spectra those of their
// (2n−1)² x-windows (full 2n−1 rows staged, 4 channels per CTA for the larger band).
// BB: block size (b = n, or b = 16 − n on the P = 15 grid for 3 ≤ n ≤ 7, R18; windows
// keep b = n)
template <int NN, bool WIN = false, int BB = NN>
__global__ void __launch_bounds__(128) oaa_tile_spectra_kernel(const TileSpecParams p) {
  static_assert(!WIN || BB == NN, "windows are for blocks of the kernel's size");
  constexpr int P = BB + NN - 1, H = (P + 1) / 2, CG = WIN ? 4 : 16, QGL = WIN ? 0 : 2, ROWS = WIN ? P : BB;
  extern __shared__ __align__(16) float band[];  // [CG][ROWS][BW] (channel stride CSTR)
  __shared__ float2 tw[16];
  const int tid = threadIdx.x, nthr = blockDim.x;
  if (tid < P) {
    float sn, cs;
    sincospif(2.0f * (float)tid / (float)P, &sn, &cs);
    tw[tid] = make_float2(cs, sn);
  }
  const int item = blockIdx.x;
  const int bl = item / p.T, t1 = item - (item / p.T) * p.T;
  const int b = p.b0 + bl;
  const int bt0 = (bl * p.T + t1) * p.T;
  const int Cinp = (p.Cin + 3) & ~3;
  const int TH8 = (p.T + 7) >> 3;
  const float* in_b = p.in + (size_t)b * p.Cin * p.R * p.R;
  // one channel group of CG per CTA (blockIdx.y; the last group also zeroes the K padding):
  // items × groups CTAs keep more of them in flight than a channel loop inside the CTA
  {
    const int c0 = blockIdx.y * CG;
    const int ncg = min(CG, p.Cin - c0);
    const int lane = tid & 31, warp = tid >> 5, nwarps = nthr >> 5;
    const int org = WIN ? p.org : 0;
    for (int sgm = warp; sgm < ncg * ROWS; sgm += nwarps) {
      const int ch = sgm / ROWS, rr = sgm - (sgm / ROWS) * ROWS;
      const int r = t1 * BB + org + rr;
      const bool rok = r >= 0 && r < p.R;
      const int roff = ((c0 + ch) * p.R + (rok ? r : 0)) * p.R;  // within the image (32-bit)
      float* d = band + ch * p.CSTR + rr * p.BW;
      for (int q = lane; q < p.BW; q += 32) {
        const int col = q + org;
        const bool ok = rok && col >= 0 && col < p.R;
        cp_async4(d + q, in_b + (ok ? roff + col : 0), ok);
      }
    }
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();
    // task u: 8 consecutive tiles (u & 7) × the CTA's channel quads × (f1, tile octet)
    const int ntask = (H * TH8 * 8) << QGL;
    for (int u = tid; u < ntask; u += nthr) {
      const int rest = u >> (3 + QGL);
      const int t2 = (rest % TH8) * 8 + (u & 7), cq = (u >> 3) & ((1 << QGL) - 1), f1 = rest / TH8;
      const int cb = c0 + 4 * cq;
      if (t2 >= p.T || cb >= Cinp) continue;
      float cf[ROWS], sf[ROWS];
#pragma unroll
      for (int p1 = 0; p1 < ROWS; ++p1) {
        const float2 t = tw[(f1 * p1) % P];
        cf[p1] = t.x;
        sf[p1] = t.y;
      }
      float xr[4][P], xi[4][P];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (cb + i < p.Cin) {
          if constexpr (WIN) {
            // window: column DFT over all 2n−1 rows at this f1, then the full row DFT
            const float* blk = band + (cb + i - c0) * p.CSTR + t2 * NN;
            float rr[P], ri[P];
#pragma unroll
            for (int p2 = 0; p2 < P; ++p2) { rr[p2] = blk[p2]; ri[p2] = 0.f; }
#pragma unroll
            for (int p1 = 1; p1 < P; ++p1) {
#pragma unroll
              for (int p2 = 0; p2 < P; ++p2) {
                const float v = blk[p1 * p.BW + p2];
                rr[p2] = fmaf(v, cf[p1], rr[p2]);
                ri[p2] = fmaf(-v, sf[p1], ri[p2]);
              }
            }
            dft<P, -1>(rr, ri, xr[i], xi[i]);
          } else {
            block_row_spectrum_smem<BB, P>(band + (cb + i - c0) * p.CSTR, p.BW, t2 * BB, cf, sf, xr[i], xi[i]);
          }
        } else {
#pragma unroll
          for (int f2 = 0; f2 < P; ++f2) { xr[i][f2] = 0.f; xi[i][f2] = 0.f; }
        }
      }
      const int bt = bt0 + t2;
      if (p.Ga) {
#pragma unroll
        for (int f2 = 0; f2 < P; ++f2) {
          const int f = f1 * P + f2;
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (cb + i < p.Cin)
              *reinterpret_cast<float2*>(p.Ga + tc_idx(f, p.KcG, p.RTG, cb + i, 2 * bt)) =
                  make_float2(xr[i][f2], xi[i][f2]);
        }
      }
#pragma unroll
      for (int f2 = 0; f2 < P; ++f2) {
        const int f = f1 * P + f2;
        const float4 vr = make_float4(xr[0][f2], xr[1][f2], xr[2][f2], xr[3][f2]);
        const float4 vi = make_float4(xi[0][f2], xi[1][f2], xi[2][f2], xi[3][f2]);
        if (!p.split) {
          *reinterpret_cast<float4*>(p.Xg + tc_idx(f, p.Kc, p.RTB, bt, cb)) = vr;
          *reinterpret_cast<float4*>(p.Xg + tc_idx(f, p.Kc, p.RTB, bt, Cinp + cb)) = vi;
        } else {
          auto hi4 = [](float4 v) {
            return make_float4(__uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u),
                               __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u),
                               __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u),
                               __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u));
          };
          const float4 hr = hi4(vr), hi_ = hi4(vi);
          *reinterpret_cast<float4*>(p.Xg + tc_idx_split(f, p.Kc, p.RTB, 0, bt, cb)) = hr;
          *reinterpret_cast<float4*>(p.Xg + tc_idx_split(f, p.Kc, p.RTB, 1, bt, cb)) =
              make_float4(vr.x - hr.x, vr.y - hr.y, vr.z - hr.z, vr.w - hr.w);
          *reinterpret_cast<float4*>(p.Xg + tc_idx_split(f, p.Kc, p.RTB, 0, bt, Cinp + cb)) = hi_;
          *reinterpret_cast<float4*>(p.Xg + tc_idx_split(f, p.Kc, p.RTB, 1, bt, Cinp + cb)) =
              make_float4(vi.x - hi_.x, vi.y - hi_.y, vi.z - hi_.z, vi.w - hi_.w);
        }
      }
    }
  }
  // zero the K padding columns (2·Cinp ≤ kk < 32·Kc) of this item's rows
  if (blockIdx.y != gridDim.y - 1) return;
  const int padq = (32 * p.Kc - 2 * Cinp) >> 2;
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int e = tid; e < H * P * p.T * padq; e += nthr) {
    const int qq = e % padq, rest = e / padq;
    const int t2 = rest % p.T, f = rest / p.T;
    if (!p.split) {
      *reinterpret_cast<float4*>(p.Xg + tc_idx(f, p.Kc, p.RTB, bt0 + t2, 2 * Cinp + 4 * qq)) = z;
    } else {
      *reinterpret_cast<float4*>(p.Xg + tc_idx_split(f, p.Kc, p.RTB, 0, bt0 + t2, 2 * Cinp + 4 * qq)) = z;
      *reinterpret_cast<float4*>(p.Xg + tc_idx_split(f, p.Kc, p.RTB, 1, bt0 + t2, 2 * Cinp + 4 * qq)) = z;
    }
  }
}

// Operands of the tensor-core weight gradient:
//   dŴ[f][k][c] = Σ_bt conj(Ĝ[f][k][bt])·Ξ̂[f][c][bt]
// as one real GEMM per bin with the reduction index j = 2·bt + {0: re, 1: im}:
//   A rows k      : (Gr, Gi)                       (G mode: n×n dy blocks)
//   B rows c      : (Xr, Xi)  → D[k][c]   = Re dŴ   (X mode: (2n−1)² x windows)
//   B rows C + c  : (Xi, −Xr) → D[k][C+c] = Im dŴ
// bt = (b − b0)·Td² + t1·Td + t2 over the dy blocks of a batch chunk; the x window of
// block (t1, t2) starts at (t1·n + org, t2·n + org), org = o − (n−1) (zero outside x).
struct FiltSpecParams {
  const float* src;  // dy [B][K][M][M] (G) or x [B][C][N][N] (X)
  float* Op;         // blocked [F][Kc][2][RT][4096]
  int nch, R, Td, org, b0, Kc, RT, SW;
  int nitems;        // (image, tile row) items of the chunk
  int BB;            // block size (launcher: 0 / n, or 16 − n -- DESIGN.md R18)
};

constexpr int kFsCG = 4;  // channels per CTA of oaa_filter_spectra_kernel (32·kFsCG threads)
// (n ≤ 5: capped at 80 registers for 6 CTAs / SM, AlexNet-like bwd_filter 1.55 → 1.45 ms; n = 8
// keeps its 165-205 registers: at 80 or 128 the spills cost more than the occupancy gains)
template <int NN, bool XWIN, int BB = NN>
__global__ void __launch_bounds__(32 * kFsCG, NN <= 5 ? 6 : 1) oaa_filter_spectra_kernel(const FiltSpecParams p) {
  constexpr int P = BB + NN - 1, H = (P + 1) / 2, ROWS = XWIN ? P : BB, CG = kFsCG;
  // [2][CG][ROWS][SW]: the CTA walks items blockIdx.x, blockIdx.x + gridDim.x, ... with the
  // next item's band staged (cp.async) while the current one is transformed -- small images
  // have little work per item, so the staging latency would otherwise dominate
  extern __shared__ __align__(16) float band[];
  const int tid = threadIdx.x;
  const int kl = tid % CG, grp = tid / CG;       // channel within group, lane group
  const int f1 = grp % H, tsub = grp / H, nsub = 32 / H;
  float tcx[ROWS], tsx[ROWS];  // e^{−2πi f1 p1 / P} for the column stage
#pragma unroll
  for (int p1 = 0; p1 < ROWS; ++p1) {
    float sn, cs;
    sincospif(2.0f * (float)((f1 * p1) % P) / (float)P, &sn, &cs);
    tcx[p1] = cs;
    tsx[p1] = sn;
  }
  const int plane = p.R * p.R;
  // one channel group of CG per CTA (blockIdx.y)
  const int c0 = blockIdx.y * CG;
  if (c0 >= p.nch) return;
  const int ncg = min(CG, p.nch - c0);
  const int bandf = CG * ROWS * p.SW;  // floats per band buffer
  auto stage = [&](int item, int buf) {
    if (item < p.nitems) {
      const int bl = item / p.Td, t1 = item - (item / p.Td) * p.Td;
      const int r0 = t1 * BB + p.org;
      const int lane = tid & 31, warp = tid >> 5;
      const float* base = p.src + ((size_t)(p.b0 + bl) * p.nch + c0) * plane;  // 32-bit offsets below
      for (int sg = warp; sg < ncg * ROWS; sg += CG) {
        const int ch = sg / ROWS, rr = sg - (sg / ROWS) * ROWS;
        const int r = r0 + rr;
        const bool rok = r >= 0 && r < p.R;
        const int roff = ch * plane + (rok ? r : 0) * p.R + p.org;
        float* d = band + buf * bandf + (ch * ROWS + rr) * p.SW;
        for (int q = lane; q < p.SW; q += 32) {
          const int col = q + p.org;
          const bool ok = rok && col >= 0 && col < p.R;
          cp_async4(d + q, base + (ok ? roff + q : 0), ok);
        }
      }
    }
    cp_async_commit();
  };
  stage(blockIdx.x, 0);
  int buf = 0;
  for (int item = blockIdx.x; item < p.nitems; item += gridDim.x, buf ^= 1) {
    stage(item + gridDim.x, buf ^ 1);
    asm volatile("cp.async.wait_group 1;" ::: "memory");  // this item's band has landed
    __syncthreads();
    const int bl = item / p.Td, t1 = item - (item / p.Td) * p.Td;
    const int bt0 = (bl * p.Td + t1) * p.Td;
    const int q_lo = bt0 >> 1, q_hi = (bt0 + p.Td - 1) >> 1;
    if (kl < ncg && tsub < nsub) {
      const float* bsrc = band + buf * bandf + kl * ROWS * p.SW;
      const int ch = c0 + kl;
      for (int q = q_lo + tsub; q <= q_hi; q += nsub) {
        float sr[2][P], si[2][P];
        bool have[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int bt = 2 * q + h;
          have[h] = bt >= bt0 && bt < bt0 + p.Td;
          const int t2 = have[h] ? bt - bt0 : 0;
          if constexpr (!XWIN) {
            float cf[BB], sf[BB];
#pragma unroll
            for (int p1 = 0; p1 < BB; ++p1) { cf[p1] = tcx[p1]; sf[p1] = tsx[p1]; }
            block_row_spectrum_smem<BB, P>(bsrc, p.SW, t2 * BB, cf, sf, sr[h], si[h]);
          } else {
            const float* w = bsrc + t2 * BB;
            float rr[P], ri[P];
#pragma unroll
            for (int p2 = 0; p2 < P; ++p2) {
              float a = w[p2], bb = 0.f;
#pragma unroll
              for (int p1 = 1; p1 < P; ++p1) {
                const float v = w[p1 * p.SW + p2];
                a = fmaf(v, tcx[p1], a);
                bb = fmaf(-v, tsx[p1], bb);
              }
              rr[p2] = a;
              ri[p2] = bb;
            }
            dft<P, -1>(rr, ri, sr[h], si[h]);
          }
        }
#pragma unroll
        for (int f2 = 0; f2 < P; ++f2) {
          const int f = f1 * P + f2;
          // row ch: (re, im) pairs; X mode also row nch + ch: (im, −re)
#pragma unroll
          for (int rowk = 0; rowk < (XWIN ? 2 : 1); ++rowk) {
            float v[4];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              v[2 * h] = rowk == 0 ? sr[h][f2] : si[h][f2];
              v[2 * h + 1] = rowk == 0 ? si[h][f2] : -sr[h][f2];
            }
            const int row = ch + rowk * p.nch;
            float* dh = p.Op + tc_idx(f, p.Kc, p.RT, row, 4 * q);
            if (have[0] && have[1]) {
              *reinterpret_cast<float4*>(dh) = make_float4(v[0], v[1], v[2], v[3]);
            } else if (have[0]) {
              *reinterpret_cast<float2*>(dh) = make_float2(v[0], v[1]);
            } else {
              *reinterpret_cast<float2*>(dh + 2) = make_float2(v[2], v[3]);
            }
          }
        }
      }
    }
    __syncthreads();  // every thread is done with this band before it is restaged
  }
  cp_async_wait_all();
}

#ifdef OAA_DEFINE_AUX_KERNELS
// Zero the reduction columns j ∈ [j0, j1) of every row of a blocked operand.
__global__ void oaa_tc_zero_tail_kernel(float* Op, int F, int Kc, int RT, int j0, int j1) {
  const int tail = j1 - j0;
  if (tail <= 0) return;
  const long long total = (long long)F * RT * 128 * tail;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int j = j0 + (int)(t % tail);
    const int r = (int)((t / tail) % (RT * 128));
    const int f = (int)(t / ((long long)tail * RT * 128));
    Op[tc_idx(f, Kc, RT, r, j)] = 0.f;
  }
}

#endif  // OAA_DEFINE_AUX_KERNELS

}  // namespace oaa
