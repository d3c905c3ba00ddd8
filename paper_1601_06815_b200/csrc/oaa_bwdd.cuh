// oaa_bwdd.cuh -- bwd_data for layers with few input channels (C ≤ 4): the first of the
// two backward convolutions of PAPER.md:89, dx = crop(Σ_k FullConv(dy_k, flip180 w_kc)),
// evaluated by OaA over the n×n blocks of dy -- or, for 3 ≤ n ≤ 7 and
// large images, over b×b blocks with b = 16 − n on the P = 15 grid (R18); with b ≥ n − 1
// the vertical overlap still gives each dx element at most two addends (below).
//
// One CTA per (image b, dy tile row t1).  Compute warp i owns chunk i of the tile row:
// lanes (tt, f1) hold block t2 = i·TPW + tt, spectrum row f1.  For every dy channel k in
// turn each warp stages the n dy rows of its own columns (cp.async, zero padded, 8-deep
// per-warp ring); the k-th slice of the flipped-kernel spectra comes from a 16-deep
// shared ring of bulk copies that the last warp to release a stage refills, so warps never
// meet at a CTA barrier inside the k loop.  Per k a lane computes its block-row spectrum Ĝ_k[f1,:] (pruned column DFT +
// row codelet) and accumulates the C output spectra Ŷ_c += Ŵᶠ_{k,c}·Ĝ_k in registers.
// Epilogue per output channel c: inverse DFT along f2 (stage A, lanes (tile, f1)) → Q in
// shared memory → stage B (lanes = full-frame columns: the two block columns summed
// before the Hermitian c2r along f1, as in the walker) → overlap-add into dx.
//
// The vertical overlap (n−1 rows shared by consecutive tile rows) crosses
// CTAs: every value is added to dx (zeroed by the caller's launch sequence) with a
// fire-and-forget red.global.add.f32.  Each dx element receives at most two addends onto
// an exact zero and IEEE addition is commutative, so the result is bitwise deterministic
// whatever order the two CTAs reach it in.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "dft.cuh"
#include "oaa_kernels.cuh"
#include "oaa_walk.cuh"

namespace oaa {

struct BwdDParams {
  const float* dy;     // [B][K][M][M]
  const float4* spec;  // [K][C][P2][H] float4: DFT_P(flip180 w_kc)/P² (oaa_spectrum_kernel, flip, loop over k)
  float* dx;           // [B][C][N][N], zero on entry
  int B, K, C, M, N, Td, off;  // off = n−1−o: full-frame column/row of dx element 0
  int NCW;                     // chunk warps per tile row
  int RPC;                     // (image, tile row) pairs per CTA: RPC·NCW ≤ 8 compute warps
  int WSL;                     // log2 of the Ŵ ring depth (≤ kBwddWStages)
  int BB;                      // dy block size b (n, or 16 − n: the launcher picks the instantiation)
};

constexpr int kBwddStages = 8;    // per-warp dy ring depth (covers HBM latency)
constexpr int kBwddWStages = 16;  // max shared Ŵ ring depth: how far the fastest warp may run ahead
// dy ring depth for blocks b: 8 slices of n = b rows, 4 of the larger b = 16 − n (more
// bytes per slice; the ring then still holds more bytes in flight than at n = 8)
__host__ __device__ constexpr int bwdd_stages(int n, int bb) { return bb > n ? 4 : kBwddStages; }
// geometry of WalkGeo<n, bb>: H = (b + n) / 2 spectrum rows, TPW = 32 / H blocks per warp
__host__ __device__ constexpr int bwdd_h(int n, int bb) { return (bb + n) / 2; }
__host__ __device__ constexpr size_t bwdd_dy_bytes(int n, int bb, int NCW, int RPC) {
  return (size_t)RPC * NCW * bwdd_stages(n, bb) * bb * ((32 / bwdd_h(n, bb)) * bb) * 4;
}
__host__ __device__ constexpr size_t bwdd_q_bytes(int n, int bb, int NCW, int RPC) {
  return (size_t)RPC * (NCW * (32 / bwdd_h(n, bb)) + 1) * bwdd_h(n, bb) * (bb + n - 1) * 8;
}
// bytes of one Ŵ ring stage ([C][H][H] float4, padded to 128 B)
__host__ __device__ constexpr int bwdd_w_bytes(int n, int bb, int C) {
  return (C * bwdd_h(n, bb) * bwdd_h(n, bb) * 16 + 127) & ~127;
}
// Ŵ ring | dy ring (the epilogue's Q buffer reuses the dy ring: the k loop is over by then)
__host__ __device__ constexpr size_t bwdd_smem_bytes(int n, int bb, int C, int NCW, int RPC, int WSL) {
  return ((size_t)1 << WSL) * bwdd_w_bytes(n, bb, C) +
         (bwdd_dy_bytes(n, bb, NCW, RPC) > bwdd_q_bytes(n, bb, NCW, RPC) ? bwdd_dy_bytes(n, bb, NCW, RPC)
                                                                          : bwdd_q_bytes(n, bb, NCW, RPC));
}

__device__ __forceinline__ void cp_async_mbar_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Shared memory: Ŵ ring [kBwddWStages][C][P2][H] float4 (bulk copies, refilled by the last
// warp to release a stage) | per-warp dy ring [RPC·NCW][kBwddStages][n][CW] floats (each warp
// stages the n rows of its own CW columns); the epilogue's Q [RPC][(NCW·TPW + 1) tiles][H][P]
// float2 (last tile of each pair zero) reuses the dy ring.
// A CTA covers RPC consecutive (image, tile row) pairs (narrow images: several tile rows
// or images per CTA, so that every CTA has up to 8 compute warps sharing one Ŵ ring);
// compute warp w works on pair w / NCW, chunk w mod NCW.
// TM = true: the C output spectra are accumulated in tensor memory (96 columns per warp)
// instead of registers, so the kernel fits 128 registers and two CTAs share an SM.
// BB: dy block size b (WalkGeo; b = n is the paper's OaA, b = 16 − n the P = 15 grid)
template <int NN, int CR, bool TM = false, int BB = NN>
__device__ __forceinline__ void bwdd_body(const BwdDParams& p, const int item) {
  using G = WalkGeo<NN, BB>;
  constexpr int P = G::P, H = G::H, P2 = G::P2, TPW = G::TPW, QT = G::QT, CW = G::CW;
  constexpr int S = bwdd_stages(NN, BB);
  constexpr int DYS = BB * CW;                // floats per warp stage
  const int SW = 1 << p.WSL, SWM = SW - 1;    // Ŵ ring depth (power of two)
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ uint64_t wfull[kBwddWStages];
  __shared__ int wrel[kBwddWStages];
  __shared__ uint32_t s_tmem;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NCW = p.NCW, NCWT = p.RPC * p.NCW;  // chunk warps per pair, compute warps
  const int npairs = p.B * p.Td;
  const int wpair = warp / NCW, wchunk = warp - (warp / NCW) * NCW;  // this warp's pair, chunk
  const int pair = item * p.RPC + wpair;
  const bool pair_ok = pair < npairs;
  const int b = pair_ok ? pair / p.Td : 0, t1 = pair_ok ? pair - (pair / p.Td) * p.Td : 0;
  const int w4 = p.C * P2 * H;                // float4 of kernel spectra per dy channel
  const int wst = bwdd_w_bytes(NN, BB, p.C);  // bytes per Ŵ stage
  unsigned char* Wring = smem_raw;
  float* dyring = reinterpret_cast<float*>(smem_raw + (size_t)SW * wst);
  const uint32_t wbytes = (uint32_t)w4 * 16u;
  // Ŵ ring: stage k % SW holds the kernel spectra of dy channel k, brought in by a bulk
  // copy (TMA engine) whose completion is counted on wfull; the last warp to release a
  // stage issues the copy that refills it, so no warp ever waits for another to issue.
  if (tid == 0) {
    for (int s = 0; s < SW; ++s) {
      mbar_init(&wfull[s], 1);
      wrel[s] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  float2* Q = reinterpret_cast<float2*>(dyring);  // epilogue only (aliases the dy ring)
  const int ntile_q = NCW * TPW;  // tiles of one pair held in Q; tile ntile_q is its zero tile

  if (TM && warp == 0) {
    // warps w < 4 use columns [0, 128): narrow tile rows (≤ 4 chunk warps, N ≲ 128) take half
    // the columns, so up to 4 CTAs share an SM's 512
    if (NCWT <= 4)
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&s_tmem)));
    else
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0) {
    for (int k = 0; k < SW && k < p.K; ++k) {
      mbar_expect_tx(&wfull[k], wbytes);
      bulk_g2s(Wring + (size_t)k * wst, p.spec + (size_t)k * w4, wbytes, &wfull[k]);
    }
  }
  // a CTA of 7 chunks is launched with one extra, idle warp (both CTAs of an SM then put
  // exactly two warps on each SMSP)
  if (warp >= NCWT) return;
  auto w_wait = [&](int k) { mbar_wait(&wfull[k & SWM], (k >> p.WSL) & 1); };
  auto w_release = [&](int k) {  // after __syncwarp: this warp is done with stage k % SW
    if (lane == 0) {
      // no membar here: it would also wait for this lane's in-flight dy cp.asyncs.  The
      // warp's reads of the stage are complete (their values were consumed before the
      // __syncwarp), and the atomic orders the warps' releases.
      const int s = k & SWM;
      int old;
      asm volatile("atom.shared.inc.u32 %0, [%1], %2;" : "=r"(old) : "r"(smem_u32(&wrel[s])), "r"(NCWT - 1) : "memory");
      if (old == NCWT - 1 && k + SW < p.K) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&wfull[s], wbytes);
        bulk_g2s(Wring + (size_t)s * wst, p.spec + (size_t)(k + SW) * w4, wbytes, &wfull[s]);
      }
    }
  };
  // compute warp w: TMEM lanes 32·(w mod 4).., columns 128·(w / 4) + 32·c
  const uint32_t tacc = TM ? s_tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(warp >> 2) * 128u : 0u;

  // ---------------- compute warps: each stages its own columns of the b dy rows
  // (CW > 32 for the larger blocks: a lane stages columns lane, lane + 32)
  constexpr int NCR = (CW + 31) / 32;
  const size_t planeM = (size_t)p.M * p.M;
  int nrow = p.M - t1 * BB;                             // dy rows of this tile row inside dy
  nrow = nrow < BB ? nrow : BB;
  const float* srcb = p.dy + (size_t)b * p.K * planeM + (size_t)(t1 * BB) * p.M;
  float* mydy = dyring + (size_t)warp * S * DYS;
  auto stage_dy = [&](int k) {
#pragma unroll
    for (int cr = 0; cr < NCR; ++cr) {
      const int cl = lane + 32 * cr;                    // column of the chunk
      const int col = wchunk * CW + cl;
      const bool cok = pair_ok && cl < CW && col < p.M;
      if (k < p.K && cl < CW) {
        const float* src = srcb + (cok ? col : 0) + (size_t)k * planeM;
        float* d = mydy + (k % S) * DYS + cl;
        if (cok && nrow == BB) {
#pragma unroll
          for (int rr = 0; rr < BB; ++rr) {
            cp_async4(d, src, true);
            src += p.M;
            d += CW;
          }
        } else {
#pragma unroll
          for (int rr = 0; rr < BB; ++rr) {
            const bool ok = cok && rr < nrow;
            cp_async4(d, ok ? src : p.dy, ok);
            src += p.M;
            d += CW;
          }
        }
      }
    }
    cp_async_commit();
  };
#pragma unroll
  for (int k = 0; k < S - 2; ++k) stage_dy(k);

  const int tt = lane / H, f1 = lane - (lane / H) * H;
  const bool laneA = tt < TPW;
  const int t2 = wchunk * TPW + tt;
  float cf[BB], sf[BB];
#pragma unroll
  for (int p1 = 0; p1 < BB; ++p1) {
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

  // TM: acc[c] row in TMEM (re at columns f, im at 16 + f) += Ŵᶠ·Ĝ; warp-collective
  auto accum_tm = [&](int k, const float (&gr)[P], const float (&gi)[P]) {
    const float4* W = reinterpret_cast<const float4*>(Wring + (size_t)(k & SWM) * wst) + f1;
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
          const float4 w = W[(c * P2 + q) * H];
          const int f = 2 * q;
          a[f] = fmaf(w.x, gr[f], a[f]);
          a[f] = fmaf(-w.y, gi[f], a[f]);
          a[16 + f] = fmaf(w.x, gi[f], a[16 + f]);
          a[16 + f] = fmaf(w.y, gr[f], a[16 + f]);
          if (f + 1 < P) {
            a[f + 1] = fmaf(w.z, gr[f + 1], a[f + 1]);
            a[f + 1] = fmaf(-w.w, gi[f + 1], a[f + 1]);
            a[17 + f] = fmaf(w.z, gi[f + 1], a[17 + f]);
            a[17 + f] = fmaf(w.w, gr[f + 1], a[17 + f]);
          }
        }
        tm_st32(tacc + 32 * c, a);
      }
    }
  };
  auto accum = [&](int k, const float (&gr)[P], const float (&gi)[P]) {
    const float4* W = reinterpret_cast<const float4*>(Wring + (size_t)(k & SWM) * wst) + f1;
#pragma unroll
    for (int c = 0; c < CR; ++c) {
      if (c < p.C) {
#pragma unroll
        for (int q = 0; q < P2; ++q) {
          const float4 w = W[(c * P2 + q) * H];
          const int f = 2 * q;
          ar[c][f] = fmaf(w.x, gr[f], ar[c][f]);
          ar[c][f] = fmaf(-w.y, gi[f], ar[c][f]);
          ai[c][f] = fmaf(w.x, gi[f], ai[c][f]);
          ai[c][f] = fmaf(w.y, gr[f], ai[c][f]);
          if (f + 1 < P) {
            ar[c][f + 1] = fmaf(w.z, gr[f + 1], ar[c][f + 1]);
            ar[c][f + 1] = fmaf(-w.w, gi[f + 1], ar[c][f + 1]);
            ai[c][f + 1] = fmaf(w.z, gi[f + 1], ai[c][f + 1]);
            ai[c][f + 1] = fmaf(w.w, gr[f + 1], ai[c][f + 1]);
          }
        }
      }
    }
  };
  // two dy channels per step: their block transforms are independent (ILP); the
  // prefetch distance is S − 2 so the two refilled stages are the ones just consumed
  int k = 0;
  if constexpr (TM) {
    // one channel per step (register budget); the ring prefetch distance stays S − 2
    for (; k < p.K; ++k) {
      const int s0 = k % S;
      stage_dy(k + S - 2);
      asm volatile("cp.async.wait_group %0;" ::"n"(S - 2) : "memory");
      __syncwarp();
      w_wait(k);
      float gr[P], gi[P];
      block_row_spectrum_smem<BB, P>(mydy + s0 * DYS, CW, (laneA ? tt : 0) * BB, cf, sf, gr, gi);
      accum_tm(k, gr, gi);
      __syncwarp();
      w_release(k);
    }
  }
  for (; k + 1 < p.K; k += 2) {
    const int s0 = k % S, s1 = (k + 1) % S;
    stage_dy(k + S - 2);
    stage_dy(k + S - 1);
    asm volatile("cp.async.wait_group %0;" ::"n"(S - 2) : "memory");  // groups k, k+1 landed
    __syncwarp();
    w_wait(k);
    w_wait(k + 1);
    if (laneA) {
      float g0r[P], g0i[P], g1r[P], g1i[P];
      block_row_spectrum_smem<BB, P>(mydy + s0 * DYS, CW, tt * BB, cf, sf, g0r, g0i);
      block_row_spectrum_smem<BB, P>(mydy + s1 * DYS, CW, tt * BB, cf, sf, g1r, g1i);
      accum(k, g0r, g0i);
      accum(k + 1, g1r, g1i);
    }
    __syncwarp();
    w_release(k);
    w_release(k + 1);
  }
  if (k < p.K) {  // odd K: last channel
    const int s0 = k % S;
    cp_async_wait_all();
    __syncwarp();
    w_wait(k);
    if (laneA) {
      float gr[P], gi[P];
      block_row_spectrum_smem<BB, P>(mydy + s0 * DYS, CW, tt * BB, cf, sf, gr, gi);
      accum(k, gr, gi);
    }
    __syncwarp();
    w_release(k);
  }
  cp_async_wait_all();

  // ---------------- epilogue: per output channel, inverse DFT + overlap-add into dx
  const int nthr_c = 32 * NCWT;
  // Q reuses the dy ring: every compute warp is past its last dy stage first
  asm volatile("bar.sync 1, %0;" ::"r"(nthr_c) : "memory");
  const int QP = (ntile_q + 1) * QT;  // float2 per pair in Q
  for (int e = tid; e < p.RPC * QT; e += nthr_c) {
    const int r = e / QT;
    Q[r * QP + ntile_q * QT + (e - r * QT)] = make_float2(0.f, 0.f);
  }
  const int FW = p.Td * BB + NN - 1;  // full-frame width
  const size_t planeN = (size_t)p.N * p.N;
#pragma unroll
  for (int c = 0; c < CR; ++c) {
    if (c >= p.C) break;
    asm volatile("bar.sync 1, %0;" ::"r"(nthr_c) : "memory");  // Q free
    float er[P], ei[P];
    if constexpr (TM) {
      float a[32];
      __syncwarp();
      tmem_wait_st();
      tm_ld32(tacc + 32 * c, a);
      tmem_wait_ld();
#pragma unroll
      for (int f = 0; f < P; ++f) { er[f] = a[f]; ei[f] = a[16 + f]; }
    } else {
#pragma unroll
      for (int f = 0; f < P; ++f) { er[f] = ar[c][f]; ei[f] = ai[c][f]; }
    }
    if (laneA) {
      float qr[P], qi[P];
      dft<P, +1>(er, ei, qr, qi);
      float2* qd = Q + wpair * QP + t2 * QT + f1 * P;
      const bool real_tile = pair_ok && t2 < p.Td;
#pragma unroll
      for (int p2 = 0; p2 < P; ++p2) qd[p2] = real_tile ? make_float2(qr[p2], qi[p2]) : make_float2(0.f, 0.f);
    }
    asm volatile("bar.sync 1, %0;" ::"r"(nthr_c) : "memory");  // Q complete
    for (int e = tid; e < p.RPC * FW; e += nthr_c) {
      const int r = e / FW, J = e - (e / FW) * FW;
      const int pr = item * p.RPC + r;
      const int j = J - p.off;
      if (pr >= npairs || j < 0 || j >= p.N) continue;
      const int pb = pr / p.Td, pt1 = pr - (pr / p.Td) * p.Td;
      float* dxc = p.dx + ((size_t)pb * p.C + c) * planeN;
      const int I0 = pt1 * BB - p.off;  // dx row of block row 0
      const int tA = J / BB, pA = J - (J / BB) * BB;
      const int offA = r * QP + (tA < p.Td ? tA : ntile_q) * QT + pA;
      const int offB = r * QP + ((pA <= NN - 2 && tA >= 1) ? (tA - 1) * QT + pA + BB : ntile_q * QT);
      float zr[H], zi[H];
#pragma unroll
      for (int f = 0; f < H; ++f) {
        const float2 a = Q[offA + f * P], bb = Q[offB + f * P];
        zr[f] = a.x + bb.x;
        zi[f] = a.y + bb.y;
      }
      float y[P];
      c2r_half<P>(zr, zi, y);
#pragma unroll
      for (int p1 = 0; p1 < P; ++p1) {
        const int r = I0 + p1;
        if (r >= 0 && r < p.N) atomicAdd(dxc + (size_t)r * p.N + j, y[p1]);
      }
    }
  }
  if constexpr (TM) {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    asm volatile("bar.sync 1, %0;" ::"r"(nthr_c) : "memory");
    if (warp == 0) {
      if (NCWT <= 4) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(s_tmem));
      else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(s_tmem));
    }
  }
}

template <int NN, int CR, bool TM = false, int BB = NN>
__global__ void __launch_bounds__(256, TM ? 2 : 1) oaa_bwdd_kernel(const BwdDParams p) {
  bwdd_body<NN, CR, TM, BB>(p, blockIdx.x);
}

}  // namespace oaa
