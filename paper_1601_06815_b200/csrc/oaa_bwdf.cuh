// oaa_bwdf.cuh -- bwd_filter (the second backward convolution of PAPER.md:89, the
// correlation of input and output-gradient blocks):
//   dŴ[f][k][c] = Σ_{b, dy block s} conj(Ĝ_s[k][f]) · Ξ̂_s[c][f]
// with Ĝ_s the spectrum of dy block s (n×n, zero padded to P×P) and Ξ̂_s the spectrum of
// the (2n−1)² x-window of that block (computed once per (image, block, channel) by
// oaa_xspec_kernel<n, true> into the chunked layout of oaa_walk.cuh).
//
// CTA (g, k-group): 8 warps, warp w owns KPW = ⌊32/H⌋ kernels, lanes (ks, f1), and
// accumulates the lane's dŴ row f1 for all C channels in registers over a static,
// deterministic slice of the (image, dy tile row) items (item = g + j·G).  Per chunk of
// TPW dy blocks:
//   * Ξ̂ of the chunk arrives in a shared ring by bulk copy (TMA engine); the last warp to
//     release a slot refills it (as in the walker), no producer warp, no CTA barrier;
//   * each warp stages the n dy rows × CW columns of its KPW kernels itself (cp.async,
//     per-warp ring), so warps never wait for each other;
//   * per block: Ĝ row f1 (pruned column DFT + row codelet), then the C complex MACs.
// Partial spectra go to partial[g][k][c][f2][f1]; oaa_filter_finalize_kernel sums the G
// slices in fp64 (fixed order), inverse-transforms and reads the lags.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "dft.cuh"
#include "oaa_kernels.cuh"
#include "oaa_walk.cuh"
#include "oaa_bwdd.cuh"

namespace oaa {

struct BwdFParams {
  const float* dy;    // [B][K][M][M]
  const float4* XS;   // Ξ̂ chunks [B·Td][NCH][C][32][RS4]
  float2* partial;    // [G][K][C][P][H]
  int B, K, C, M, Td, NCH, G;
  int KG;             // kernels per CTA (a multiple of ⌊32/n⌋; blockDim = 32·KG/⌊32/n⌋)
};

constexpr int kBwdfWarps = 8;
// TM = false: dŴ accumulators in registers (small n: C·P complex values per lane);
// TM = true : accumulators in tensor memory (every block: a 32-column ld + st per channel).
// Both ≤ 128 registers, 2 CTAs / SM.
template <bool TM> struct BwdfCfg;
template <> struct BwdfCfg<false> { static constexpr int ring = 3, dy = 2, minb = 2; };
template <> struct BwdfCfg<true> { static constexpr int ring = 3, dy = 2, minb = 2; };

template <bool TM>
__host__ __device__ constexpr size_t bwdf_smem_bytes(int n, int C) {
  return (size_t)BwdfCfg<TM>::ring * C * ((32 / n) * n * (n | 1)) * 16 +
         (size_t)kBwdfWarps * BwdfCfg<TM>::dy * (32 / n) * (n * ((32 / n) * n) + 4) * 4;
}

// g: slice of the (image, tile row) items; kgrp: kernel group; nw: warps in the CTA
template <int NN, int CR, bool TM>
__device__ __forceinline__ void bwdf_body(const BwdFParams& p, const int g, const int kgrp, const int nw) {
  constexpr int kBwdfRing = BwdfCfg<TM>::ring, kBwdfDy = BwdfCfg<TM>::dy;
  using G = WalkGeo<NN>;
  constexpr int P = G::P, H = G::H, P2 = G::P2, TPW = G::TPW, CW = G::CW, RS4 = G::RS4;
  constexpr int KPW = 32 / H;                 // kernels per warp
  // floats per kernel in a dy stage: the n×CW rows + 4 floats of padding, so the KPW
  // kernels a warp reads at the same block position hit different banks
  constexpr int KSTR = NN * CW + 4;
  constexpr int DYS = KPW * KSTR;             // floats per warp dy stage
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ uint64_t full[kBwdfRing];
  __shared__ int rel[kBwdfRing];
  __shared__ uint32_t s_tmem;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int slot4 = p.C * G::CH4;
  float4* ring = reinterpret_cast<float4*>(smem_raw);
  float* dyr = reinterpret_cast<float*>(ring + kBwdfRing * slot4) + (size_t)warp * kBwdfDy * DYS;
  const int nitems_all = p.B * p.Td;
  const int nitems = g < nitems_all ? (nitems_all - g + p.G - 1) / p.G : 0;
  const int nseq = nitems * p.NCH;
  const uint32_t slot_bytes = (uint32_t)slot4 * 16u;
  auto seq_src = [&](int sq) {
    const int j = sq / p.NCH, i = sq - (sq / p.NCH) * p.NCH;
    return p.XS + ((size_t)(g + j * p.G) * p.NCH + i) * slot4;
  };
  if (tid == 0) {
    for (int s = 0; s < kBwdfRing; ++s) {
      mbar_init(&full[s], 1);
      rel[s] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (TM && warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // warp w: TMEM lanes 32·(w mod 4).., columns 128·(w / 4) + 32·c (c < CR ≤ 4)
  const uint32_t tacc = TM ? s_tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(warp >> 2) * 128u : 0u;
  if (tid == 0) {
    for (int s = 0; s < kBwdfRing && s < nseq; ++s) {
      mbar_expect_tx(&full[s], slot_bytes);
      bulk_g2s(ring + s * slot4, seq_src(s), slot_bytes, &full[s]);
    }
  }

  const int ks = lane / H, f1 = lane - (lane / H) * H;
  const int kbase = kgrp * p.KG + warp * KPW;
  const int k = kbase + ks;
  const bool laneK = ks < KPW && k < p.K;
  float cf[NN], sf[NN];
#pragma unroll
  for (int p1 = 0; p1 < NN; ++p1) {
    float s, c;
    sincospif(2.0f * (float)((f1 * p1) % P) / (float)P, &s, &c);
    cf[p1] = c;
    sf[p1] = s;
  }
  float ar[TM ? 1 : CR][P], ai[TM ? 1 : CR][P];
  if constexpr (!TM) {
#pragma unroll
    for (int c = 0; c < CR; ++c)
#pragma unroll
      for (int f = 0; f < P; ++f) { ar[c][f] = 0.f; ai[c][f] = 0.f; }
  } else {
    float z[32];
#pragma unroll
    for (int q = 0; q < 32; ++q) z[q] = 0.f;
#pragma unroll
    for (int c = 0; c < CR; ++c) tm_st32(tacc + 32 * c, z);
  }

  // this warp's dy rows of chunk sq: rows (kernel kk, block row rr) × CW columns
  const size_t planeM = (size_t)p.M * p.M;
  auto stage_dy = [&](int sq) {
    if (sq < nseq && lane < CW) {
      const int j = sq / p.NCH, i = sq - (sq / p.NCH) * p.NCH;
      const int item = g + j * p.G;
      const int b = item / p.Td, t1 = item - (item / p.Td) * p.Td;
      const int col = i * CW + lane;
      const bool cok = col < p.M;
      int nrow = p.M - t1 * NN;
      nrow = nrow < NN ? nrow : NN;
      float* d = dyr + (sq % kBwdfDy) * DYS + lane;
      const float* src = p.dy + ((size_t)b * p.K + kbase) * planeM + (size_t)(t1 * NN) * p.M + (cok ? col : 0);
      const int nk = min(KPW, p.K - kbase);
      const ptrdiff_t kstep = (ptrdiff_t)planeM - (ptrdiff_t)NN * p.M;
      if (cok && nk == KPW && nrow == NN) {  // interior: no predicates
#pragma unroll
        for (int kk = 0; kk < KPW; ++kk) {
#pragma unroll
          for (int rr = 0; rr < NN; ++rr) {
            cp_async4(d, src, true);
            src += p.M;
            d += CW;
          }
          src += kstep;
          d += KSTR - NN * CW;
        }
      } else {
#pragma unroll
        for (int kk = 0; kk < KPW; ++kk) {
          const bool kok = cok && kk < nk;
#pragma unroll
          for (int rr = 0; rr < NN; ++rr) {
            const bool ok = kok && rr < nrow;
            cp_async4(d, ok ? src : p.dy, ok);
            src += p.M;
            d += CW;
          }
          src += kstep;
          d += KSTR - NN * CW;
        }
      }
    }
    cp_async_commit();
  };
#pragma unroll
  for (int sq = 0; sq < kBwdfDy - 1; ++sq) stage_dy(sq);

  for (int sq = 0; sq < nseq; ++sq) {
    const int s = sq % kBwdfRing;
    stage_dy(sq + kBwdfDy - 1);
    asm volatile("cp.async.wait_group %0;" ::"n"(kBwdfDy - 1) : "memory");
    __syncwarp();
    mbar_wait(&full[s], (sq / kBwdfRing) & 1);
    if (laneK) {
      const float* db = dyr + (sq % kBwdfDy) * DYS + ks * KSTR;
      const float4* xs = ring + s * slot4 + f1 * RS4;
      // two blocks per step: independent transforms interleave (ILP)
      auto accum = [&](int tt, const float (&gr)[P], const float (&gi)[P]) {
        if constexpr (TM) return;
        const float4* xt = xs + tt * H * RS4;
#pragma unroll
        for (int c = 0; c < CR; ++c) {
          if (c < p.C) {
#pragma unroll
            for (int q = 0; q < P2; ++q) {
              const float4 X = xt[c * G::CH4 + q];
              const int f = 2 * q;
              ar[c][f] = fmaf(gr[f], X.x, ar[c][f]);
              ar[c][f] = fmaf(gi[f], X.y, ar[c][f]);
              ai[c][f] = fmaf(gr[f], X.y, ai[c][f]);
              ai[c][f] = fmaf(-gi[f], X.x, ai[c][f]);
              if (f + 1 < P) {
                ar[c][f + 1] = fmaf(gr[f + 1], X.z, ar[c][f + 1]);
                ar[c][f + 1] = fmaf(gi[f + 1], X.w, ar[c][f + 1]);
                ai[c][f + 1] = fmaf(gr[f + 1], X.w, ai[c][f + 1]);
                ai[c][f + 1] = fmaf(-gi[f + 1], X.z, ai[c][f + 1]);
              }
            }
          }
        }
      };
      int tt = 0;
      if constexpr (TM) tt = TPW;  // (TM: the block loop below, outside the lane predicate)
#pragma unroll 1
      for (; tt + 1 < TPW; tt += 2) {
        float g0r[P], g0i[P], g1r[P], g1i[P];
        block_row_spectrum_smem<NN>(db, CW, tt * NN, cf, sf, g0r, g0i);
        block_row_spectrum_smem<NN>(db, CW, (tt + 1) * NN, cf, sf, g1r, g1i);
        accum(tt, g0r, g0i);
        accum(tt + 1, g1r, g1i);
      }
      if (tt < TPW) {
        float gr[P], gi[P];
        block_row_spectrum_smem<NN>(db, CW, tt * NN, cf, sf, gr, gi);
        accum(tt, gr, gi);
      }
    }
    if constexpr (TM) {
      // dŴ row in TMEM: per block, Ĝ row (registers) then per channel ld → MACs → st
      const float* db = dyr + (sq % kBwdfDy) * DYS + (laneK ? ks : 0) * KSTR;
      const float4* xs = ring + s * slot4 + f1 * RS4;
#pragma unroll 1
      for (int tt = 0; tt < TPW; ++tt) {
        float gr[P], gi[P];
        block_row_spectrum_smem<NN>(db, CW, tt * NN, cf, sf, gr, gi);
        const float4* xt = xs + tt * H * RS4;
        __syncwarp();
        tmem_wait_st();
#pragma unroll
        for (int c = 0; c < CR; ++c) {
          if (c < p.C) {
            float a[32];
            tm_ld32(tacc + 32 * c, a);
            tmem_wait_ld();
#pragma unroll
            for (int q = 0; q < P2; ++q) {
              const float4 X = xt[c * G::CH4 + q];
              const int f = 2 * q;
              a[f] = fmaf(gr[f], X.x, a[f]);
              a[f] = fmaf(gi[f], X.y, a[f]);
              a[16 + f] = fmaf(gr[f], X.y, a[16 + f]);
              a[16 + f] = fmaf(-gi[f], X.x, a[16 + f]);
              if (f + 1 < P) {
                a[f + 1] = fmaf(gr[f + 1], X.z, a[f + 1]);
                a[f + 1] = fmaf(gi[f + 1], X.w, a[f + 1]);
                a[17 + f] = fmaf(gr[f + 1], X.w, a[17 + f]);
                a[17 + f] = fmaf(-gi[f + 1], X.z, a[17 + f]);
              }
            }
            tm_st32(tacc + 32 * c, a);
          }
        }
      }
    }
    // release the Ξ̂ slot; the last warp out refills it
    __syncwarp();
    if (lane == 0) {
      // (no membar: it would also wait for this lane's in-flight dy cp.asyncs; the warp's
      // reads of the slot are complete and the atomic orders the releases)
      int old;  // inc wraps to 0 after the nw-th arrival
      asm volatile("atom.shared.inc.u32 %0, [%1], %2;" : "=r"(old) : "r"(smem_u32(&rel[s])), "r"(nw - 1) : "memory");
      if (old == nw - 1) {
        const int nx = sq + kBwdfRing;
        if (nx < nseq) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_expect_tx(&full[s], slot_bytes);
          bulk_g2s(ring + s * slot4, seq_src(nx), slot_bytes, &full[s]);
        }
      }
    }
  }
  cp_async_wait_all();
  if constexpr (TM) {
    __syncwarp();
    tmem_wait_st();
#pragma unroll
    for (int c = 0; c < CR; ++c) {
      if (c < p.C) {
        float a[32];
        tm_ld32(tacc + 32 * c, a);
        tmem_wait_ld();
        if (laneK) {
          float2* dst = p.partial + ((((size_t)g * p.K + k) * p.C + c) * P) * H + f1;
#pragma unroll
          for (int f2 = 0; f2 < P; ++f2) dst[f2 * H] = make_float2(a[f2], a[16 + f2]);
        }
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(s_tmem));
  } else if (laneK) {
#pragma unroll
    for (int c = 0; c < CR; ++c) {
      if (c < p.C) {
        float2* dst = p.partial + ((((size_t)g * p.K + k) * p.C + c) * P) * H + f1;
#pragma unroll
        for (int f2 = 0; f2 < P; ++f2) dst[f2 * H] = make_float2(ar[c][f2], ai[c][f2]);
      }
    }
  }
}

template <int NN, int CR, bool TM>
__global__ void __launch_bounds__(32 * kBwdfWarps, BwdfCfg<TM>::minb) oaa_bwdf_kernel(const BwdFParams p) {
  bwdf_body<NN, CR, TM>(p, blockIdx.x, blockIdx.y, blockDim.x >> 5);  // ≤ kBwdfWarps warps
}

// Fused backward, SIMT family (C ≤ 4; oaa_conv_bwd, NEXT-1): the two backward convolutions
// of PAPER.md:89 in ONE launch.  CTAs [0, nf) run the weight-gradient body (persistent
// slices, ~one per SM), the rest the data-gradient body, so every SM co-runs one CTA of
// each: the two bodies stress different pipes (bwd_filter TMEM + ring reads, bwd_data
// the FMA pipe) and fill each other's issue gaps.  Both bodies fit 128 registers and
// 256 TMEM columns, so two CTAs share an SM.
// BB: the data-gradient body's dy block size (b = n, or 16 − n as the stand-alone bwd_data)
template <int NN, int CR, int BB = NN>
__global__ void __launch_bounds__(256, 2) oaa_bwd_fused_kernel(const BwdDParams pd, const BwdFParams pf, int nf,
                                                                int G) {
  const int c = blockIdx.x;
  if (c < nf) bwdf_body<NN, CR, true>(pf, c % G, c / G, kBwdfWarps);
  else bwdd_body<NN, CR, true, BB>(pd, c - nf);
}

}  // namespace oaa
