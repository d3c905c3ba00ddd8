// oaa_tc.cuh -- tensor-core (tcgen05, sm_100a) per-frequency-bin complex channel
// contraction for layers with many channels ("genuinely dense
// contraction ... on tensor cores"; PAPER.md:15 the K·C convolutions of a layer).
//
// For every bin f the contraction Ŷ_f = Ŵ_f · X̂_f (K×C complex by C×B·T complex) is
// real-ified,
//      [Yr; Yi] (2K × N) = [[Wr, −Wi], [Wi, Wr]] (2K × 2C) · [Xr; Xi] (2C × N),
// and evaluated as D[f] = A[f] · B[f]ᵀ (A[f] M×Kd, B[f] N×Kd, both K-major).  fp32
// accuracy (rel-L2 ≤ 1e-5, R9) needs 3×TF32: every operand is split
// x = hi + lo (hi = x with the low 13 mantissa bits cleared, lo = x − hi) and
// D = A_lo·B_hi + A_hi·B_lo + A_hi·B_hi accumulates in tensor memory.
//
// Operands arrive as plain fp32 in the UMMA-blocked layout written by their producers
// (tile spectra / real-ified weights, oaa_kernels.cuh): for each (bin, 32-wide K chunk)
// the row tiles of 128 rows are consecutive 16 KB blocks in the canonical no-swizzle
// K-major order (8-row × 16-byte core matrices: LBO = 128 B between the two K halves of an
// MMA, SBO = 1 KB between 8-row groups).  Every pipeline stage is two bulk copies
// (cp.async.bulk, TMA engine); two converter warps split the stage in shared memory (hi in
// place, lo into the stage's second half), so HBM carries each operand once.
//
// Kernel (one CTA = one 128 × 256 output tile of one bin, 128 threads, 1 CTA/SM):
//   * warp 0 lane 0: producer -- per K chunk waits for the stage to be free, posts the
//     byte count on the stage's "full" mbarrier and issues the bulk copies;
//   * warp 1 lane 0: MMA issuer -- waits "full", issues 4 k-steps × 3 tcgen05.mma
//     .kind::tf32 (M=128, N=256, K=8) and commits them to the stage's "empty" mbarrier;
//   * all 4 warps: epilogue, tcgen05.ld of the 128 × 256 fp32 accumulator (thread = row).
#pragma once
#include <cuda.h>  // CUtensorMap (encoded on the host, oaa_abi.cu)
#include <cuda_runtime.h>
#include <stdint.h>

#include "oaa_kernels.cuh"

namespace oaa {

#ifdef OAA_EXP_TC_SPIN  // experiment builds only: the r1 busy-spinning waits
#define OAA_TC_WAIT mbar_wait
#else
#define OAA_TC_WAIT mbar_wait_sleep
#endif

constexpr int kTcM = 128, kTcN = 256, kTcK = 32;  // CTA tile and K chunk (fp32 elements)
constexpr int kTcStages = 2;
constexpr size_t kTcStageBytes = (size_t)(2 * kTcM + 2 * kTcN) * kTcK * sizeof(float);  // 96 KB
constexpr size_t kTcSmem = kTcStages * kTcStageBytes + 8 * 32 * 33 * sizeof(float);  // + epilogue transpose buffers

struct BinGemmParams {
  // mode 2 with dtma: TMA tensor map of D as the 5-D tensor [o][blk][ri][f][32 slots]
  // (dims {32, F, 2, blocks, Cf}); the drain warps store each 32-row × 32-slot sub-tile with
  // one cp.async.bulk.tensor from their 128-byte-swizzled shared buffer
  CUtensorMap dmap;
  int dtma;
  const float* A;  // blocked [F][Kc][2][RTA][4096]
  const float* B;  // blocked [F][Kc][2][RTB][4096]  (RTB even)
  float* D;        // [F][M][ldd] (row m, column n)
  int F, M, N, Kc, RTA, RTB, ldd;
  long long strideD;  // per-bin stride of D (elements)
  // split-K: grid.z = F·S, split s reduces K chunks [s·kps, min(Kc, (s+1)·kps))
  int S, kps;
  // mode 1 (weight gradient): instead of D, write the split's partial dŴ in the layout of
  // oaa_filter_finalize_kernel, partial[g0+s][k=m][c][f2·H+f1] (float2), columns
  // n < Cf → real part of c = n, n ≥ Cf → imaginary part of c = n − Cf.
  int mode, Cf, H, P, g0, accumulate;
  float* partial;
  int NB;  // B row tiles per CTA (1: N tile 128, 2: N tile 256); RTB is a multiple of NB
  int Kuse;  // K chunks holding data (≤ Kc; the rest of the layout is never read)
  // mode 2 (fwd / bwd_data, read by oaa_walk_kernel in load mode): column bt = (b·TT + t1)·TT
  // + t2 is walker slot s = ((b·TT + t1)·NT4 + t2 / TPW)·TPW + t2 % TPW (tile rows padded to
  // whole walker chunks of TPW tiles); row m = ri·Cf + o of bin f = f1·P + f2 goes to
  //   D[o·plane + (s / SB)·2·SB·F + ri·SB·F + f·SB + s % SB],   F = H·P bins, SB = 32 slots,
  // i.e. blocks of 32 slots: every bin's run is one aligned 128-byte line, and a walker chunk
  // spans one or two blocks
  int a_split;  // A arrives pre-split ([F][Kc][hi|lo][RTA][4096])
  int b_split;  // B arrives pre-split likewise (else the converter warps split it)
  int TT, TPW, NT4, SB, SBL;  // SB = 1 << SBL slots per block (32, oaa_walk.cuh kYSBL)
  long long plane;
};

// Instruction descriptor: D f32, A/B tf32, both K-major.
__host__ __device__ constexpr uint32_t umma_idesc_tf32(int M, int N) {
  return (1u << 4)                 // c_format = F32
         | (2u << 7)               // a_format = TF32
         | (2u << 10)              // b_format = TF32
         | (0u << 15) | (0u << 16) // K-major A and B
         | ((uint32_t)(N >> 3) << 17)
         | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void umma_tf32(uint32_t dtmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(dtmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t ta, float (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]),
        "=f"(v[8]), "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]), "=f"(v[14]), "=f"(v[15]),
        "=f"(v[16]), "=f"(v[17]), "=f"(v[18]), "=f"(v[19]), "=f"(v[20]), "=f"(v[21]), "=f"(v[22]), "=f"(v[23]),
        "=f"(v[24]), "=f"(v[25]), "=f"(v[26]), "=f"(v[27]), "=f"(v[28]), "=f"(v[29]), "=f"(v[30]), "=f"(v[31])
      : "r"(ta));
}

// K chunks accumulated in one TMEM accumulator before it is drained into registers.  The
// tensor core's fp32 accumulation truncates, so its error grows with the number of
// accumulate steps; draining every kTcDrain chunks and summing the drained values with
// round-to-nearest FADDs keeps long reductions (the weight gradient's B·T′) at fp32
// accuracy.
constexpr int kTcDrain = 8;
// warp 0 TMA producer, warp 1 MMA issuer, warps 2..9 drain/epilogue, (CONV) warps 10, 11 hi/lo
// converters.  Without CONV both operands must arrive pre-split.
template <bool CONV> constexpr int tc_threads() { return CONV ? 384 : 320; }

// D[f][m][n] = Σ_k A[f][m][k] · B[f][n][k]  (3×TF32).  grid = (ceil(N/(128·NB)), ceil(M/128), F·S)
// Two TMEM accumulators of 256 columns alternate per group of kTcDrain K chunks, so the
// MMAs of group g+1 run while the epilogue warps drain group g.
template <bool CONV>
__global__ void __launch_bounds__(tc_threads<CONV>(), 1) oaa_bin_gemm_kernel(const __grid_constant__ BinGemmParams p) {
  // Persistent: CTA b takes output tiles b, b + gridDim.x, ...  (tile order: M tiles of one
  // (bin, N tile) first, so their shared B operand is re-read from L2).  The smem stage ring
  // and the two TMEM accumulators carry on across tiles: the drain warps write tile t while
  // the MMAs of tile t+1 already run into the other accumulator.
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // stage s: [A_hi 16K][A_lo 16K][B_hi 32K][B_lo 32K]
  __shared__ uint64_t full[kTcStages], conv[kTcStages], empty[kTcStages], accf[2], acce[2];
  __shared__ uint32_t s_tmem;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int NB = p.NB, ntile = kTcM * NB;
  const bool presplit = !CONV;  // (the host launches CONV unless a_split && b_split)
  const int nN = (p.N + ntile - 1) / ntile, nM = (p.M + kTcM - 1) / kTcM;
  const int ntiles = nN * nM * p.F * p.S;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 32) {
    for (int s = 0; s < kTcStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&conv[s], 2);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&accf[b], 1);
      mbar_init(&acce[b], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s_tmem;
  constexpr uint32_t kBlk = 4096 * sizeof(float);
  struct Tile {
    int f, split, kbeg, nk, mt, nt, m0, n0, mrows, ncols, nb;
  };
  auto tile_of = [&](int t) {
    Tile T;
    const int fz = t / (nN * nM), rem = t - fz * (nN * nM);
    T.nt = rem / nM;
    T.mt = rem - T.nt * nM;
    T.f = fz / p.S;
    T.split = fz - T.f * p.S;
    T.kbeg = T.split * p.kps;
    T.nk = min(min(p.Kc, p.Kuse), T.kbeg + p.kps) - T.kbeg;
    T.m0 = T.mt * kTcM;
    T.n0 = T.nt * ntile;
    T.mrows = min(kTcM, p.M - T.m0);
    T.ncols = min(ntile, p.N - T.n0);
    T.nb = min(NB, p.RTB - NB * T.nt);
    return T;
  };
  auto groups_of = [](int nk) { return nk > 0 ? (nk + kTcDrain - 1) / kTcDrain : 0; };
  if (warp == 0) {
    if (lane == 0) {  // producer
      int gch = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const Tile T = tile_of(t);
        for (int ch = 0; ch < T.nk; ++ch, ++gch) {
          const int s = gch % kTcStages;
          if (gch >= kTcStages) OAA_TC_WAIT(&empty[s], ((gch / kTcStages) - 1) & 1);
          unsigned char* st = smem_raw + s * kTcStageBytes;
          mbar_expect_tx(&full[s], (p.a_split ? 2 : 1) * kBlk + (p.b_split ? 2 : 1) * T.nb * kBlk);
          const size_t kk = (size_t)T.f * p.Kc + T.kbeg + ch;
          const float* a = p.A + ((p.a_split ? 2 * kk : kk) * p.RTA + T.mt) * 4096;
          const float* b = p.B + ((p.b_split ? 2 * kk : kk) * p.RTB + NB * T.nt) * 4096;
          bulk_g2s(st, a, kBlk, &full[s]);
          if (p.a_split) bulk_g2s(st + kBlk, a + (size_t)p.RTA * 4096, kBlk, &full[s]);
          if (p.b_split) bulk_g2s(st + 4 * kBlk, b + (size_t)p.RTB * 4096, T.nb * kBlk, &full[s]);
          bulk_g2s(st + 2 * kBlk, b, T.nb * kBlk, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      const uint32_t idesc = NB == 2 ? umma_idesc_tf32(kTcM, 256) : umma_idesc_tf32(kTcM, 128);
      int gch = 0, gg0 = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const Tile T = tile_of(t);
        for (int ch = 0; ch < T.nk; ++ch, ++gch) {
          const int gg = gg0 + ch / kTcDrain, buf = gg & 1;
          const bool first = (ch % kTcDrain) == 0;
          if (first && gg >= 2) OAA_TC_WAIT(&acce[buf], ((gg >> 1) - 1) & 1);
          const int s = gch % kTcStages;
          OAA_TC_WAIT(presplit ? &full[s] : &conv[s], (gch / kTcStages) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t base = smem_u32(smem_raw + s * kTcStageBytes);
          const uint32_t a_hi = base, a_lo = base + kBlk, b_hi = base + 2 * kBlk, b_lo = base + 4 * kBlk;
          const uint32_t acc_t = tmem + buf * 256;
#pragma unroll
          for (int ks = 0; ks < kTcK / 8; ++ks) {  // K = 8 tf32 per MMA = 2 core-matrix columns
            const uint32_t koff = ks * 256;        // 2 × 128 B
            const uint64_t dah = umma_desc_kmajor(a_hi + koff, 128, 1024);
            const uint64_t dal = umma_desc_kmajor(a_lo + koff, 128, 1024);
            const uint64_t dbh = umma_desc_kmajor(b_hi + koff, 128, 1024);
            const uint64_t dbl = umma_desc_kmajor(b_lo + koff, 128, 1024);
#ifndef OAA_EXP_TC_NOMMA  // experiment builds only (timing): no MMAs
            umma_tf32(acc_t, dal, dbh, idesc, (first && ks == 0) ? 0u : 1u);
            umma_tf32(acc_t, dah, dbl, idesc, 1u);
            umma_tf32(acc_t, dah, dbh, idesc, 1u);
#endif
          }
          umma_commit(&empty[s]);
          if ((ch % kTcDrain) == kTcDrain - 1 || ch == T.nk - 1) umma_commit(&accf[buf]);
        }
        gg0 += groups_of(T.nk);
      }
    }
  } else if (CONV && warp >= 10) {
    // converters: x → hi (low 13 mantissa bits cleared, in place) and lo = x − hi (the
    // stage's lo slot) for the A block and the nb B blocks; the tensor core reads the
    // stage through the async proxy, hence the proxy fence before the arrive
    // (both operands pre-split: nothing to do, the MMA waits on "full" directly)
    const int ct = tid - 320;
    int gch = 0;
    for (int t = presplit ? ntiles : blockIdx.x; t < ntiles; t += gridDim.x) {
      const Tile T = tile_of(t);
      for (int ch = 0; ch < T.nk; ++ch, ++gch) {
        const int s = gch % kTcStages;
        OAA_TC_WAIT(&full[s], (gch / kTcStages) & 1);
        unsigned char* st = smem_raw + s * kTcStageBytes;
        float4* ah = reinterpret_cast<float4*>(st);
        float4* al = reinterpret_cast<float4*>(st + kBlk);
        float4* bh = reinterpret_cast<float4*>(st + 2 * kBlk);
        float4* bl = reinterpret_cast<float4*>(st + 4 * kBlk);
        const int nb4 = p.b_split ? 0 : T.nb * 1024;
        auto split4 = [](float4& h, float4& l, float4 x) {
          h.x = __uint_as_float(__float_as_uint(x.x) & 0xFFFFE000u);
          h.y = __uint_as_float(__float_as_uint(x.y) & 0xFFFFE000u);
          h.z = __uint_as_float(__float_as_uint(x.z) & 0xFFFFE000u);
          h.w = __uint_as_float(__float_as_uint(x.w) & 0xFFFFE000u);
          l = make_float4(x.x - h.x, x.y - h.y, x.z - h.z, x.w - h.w);
        };
#ifdef OAA_EXP_TC_NOCONV  // experiment builds only (timing): converters skip the split
        if (false) {
#else
        if (!p.a_split) {
#endif
#pragma unroll 4
          for (int e = ct; e < 1024; e += 64) {
            float4 h, l;
            split4(h, l, ah[e]);
            ah[e] = h;
            al[e] = l;
          }
        }
#ifdef OAA_EXP_TC_NOCONV
        for (int e = ct; e < 0; e += 64) {
#else
#pragma unroll 4
        for (int e = ct; e < nb4; e += 64) {
#endif
          float4 h, l;
          split4(h, l, bh[e]);
          bh[e] = h;
          bl[e] = l;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&conv[s]);
      }
    }
  } else {
    // drain / epilogue: warp w reads TMEM lanes 32·(w%4).., column half (w−2)/4
    const int q = warp & 3, half = (warp - 2) >> 2;
    const int row = 32 * q + lane, cb = 128 * half;
    int gg0 = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const Tile T = tile_of(t);
      const int ngroups = groups_of(T.nk);
      const bool active = cb < T.ncols;
      float acc[128];
#pragma unroll
      for (int j = 0; j < 128; ++j) acc[j] = 0.f;
      for (int gl = 0; gl < ngroups; ++gl) {
        const int gg = gg0 + gl, buf = gg & 1;
        OAA_TC_WAIT(&accf[buf], (gg >> 1) & 1);
        __syncwarp();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (active) {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            float v[32];
            tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + buf * 256 + cb + 32 * c, v);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int j = 0; j < 32; ++j) acc[32 * c + j] += v[j];
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&acce[buf]);
      }
      gg0 += ngroups;
      if (active && row < T.mrows) {
        if (p.mode == 1) {
          const int k = T.m0 + row, f1 = T.f / p.P, f2 = T.f - (T.f / p.P) * p.P;
          const int bins = p.H * p.P;
          float* pk = p.partial + ((size_t)(p.g0 + T.split) * p.M + k) * p.Cf * bins * 2 + (size_t)(f2 * p.H + f1) * 2;
#pragma unroll
          for (int j = 0; j < 128; ++j) {
            const int nn = cb + j;
            if (nn < T.ncols) {
              const int n = T.n0 + nn;
              const int im = n >= p.Cf, c = im ? n - p.Cf : n;
              float* d = pk + (size_t)c * bins * 2 + im;
              *d = p.accumulate ? *d + acc[j] : acc[j];
            }
          }
        }
      }
      if (p.mode == 2 && active && p.TT % p.TPW == 0 && p.SBL == 5) {
        // walker layout with walker slot = GEMM column (whole walker chunks per tile row):
        // a 32-column chunk of the tile is one 32-slot block, i.e. per row one 128-byte run
        // D[o·plane + blk·2·bf8 + ri·bf8 + f·32 + 0..31].  The warp's 32 rows × 32 columns go
        // through its XOR-swizzled 4 KB buffer (float4 j of row r at r·8 + (j ^ (r & 7)):
        // conflict-free both ways), then 8 lanes write each row run with 16-byte stores --
        // 4 full runs per store instruction.
        float4* tb4 = reinterpret_cast<float4*>(smem_raw + kTcStages * kTcStageBytes) + (warp - 2) * 256;
        const int nc = min(128, T.ncols - cb), nr = min(32, T.mrows - 32 * q);
        const long long bf8 = (long long)p.SB * p.H * p.P;
        const int sub = lane >> 3, ch = lane & 7;
        float* dbin = p.D + (long long)T.f * p.SB + 4 * ch;
        // rows 32q.. of the tile: one ri, o0.. (Cf a multiple of 32 for the TMA store)
        const int mg = T.m0 + 32 * q, rig = mg >= p.Cf, o0 = mg - (rig ? p.Cf : 0);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (p.dtma) {
            // the previous store of this buffer has read it
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          }
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 8; ++j)
            tb4[lane * 8 + (j ^ (lane & 7))] =
                make_float4(acc[32 * c + 4 * j], acc[32 * c + 4 * j + 1], acc[32 * c + 4 * j + 2], acc[32 * c + 4 * j + 3]);
          const int col0 = 32 * c + 4 * ch;  // tile column of this lane's 4 values
          const int blkn = (T.n0 + cb + 32 * c) >> 5;
          if (p.dtma) {
            // 128-byte swizzle of the tensor map = this buffer's XOR layout; rows past M and
            // slots past the allocation are clipped by the TMA unit
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0 && 32 * c < nc && nr > 0) {
              asm volatile(
                  "cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(
                      reinterpret_cast<uint64_t>(&p.dmap)),
                  "r"(0), "r"(T.f), "r"(rig), "r"(blkn), "r"(o0), "r"(smem_u32(tb4))
                  : "memory");
              asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            continue;
          }
          __syncwarp();
          const long long blk = (long long)blkn * 2 * bf8;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int r = 4 * i + sub;
            if (r < nr && col0 < nc) {
              const float4 v = tb4[r * 8 + (ch ^ (r & 7))];
              const int m = T.m0 + 32 * q + r, ri = m >= p.Cf;
              float* dst = dbin + (long long)(m - (ri ? p.Cf : 0)) * p.plane + (ri ? bf8 : 0) + blk;
              if (col0 + 3 < nc) {
                __stcg(reinterpret_cast<float4*>(dst), v);
              } else {
                __stcg(dst, v.x);
                if (col0 + 1 < nc) __stcg(dst + 1, v.y);
                if (col0 + 2 < nc) __stcg(dst + 2, v.z);
              }
            }
          }
        }
        if (p.dtma && lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      } else if (p.mode == 2 && active) {
        // walker layout: per bin an SB-float run of slots; transpose 32 columns at a time
        float* tb = reinterpret_cast<float*>(smem_raw + kTcStages * kTcStageBytes) + (warp - 2) * 32 * 33;
        const int nc = min(128, T.ncols - cb);
        const long long bf8 = (long long)p.SB * p.H * p.P;
        // this lane's row offset (row 32·q + lane), fetched by the storing lanes with a shuffle
        const int mrow = T.m0 + 32 * q + lane, rri = mrow >= p.Cf;
        const long long rowoff = (long long)(mrow - (rri ? p.Cf : 0)) * p.plane + (rri ? bf8 : 0);
        const int nr = min(32, T.mrows - 32 * q);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 32; ++j) tb[lane * 33 + j] = acc[32 * c + j];
          __syncwarp();
          const int col = 32 * c + lane;
          float* dcol = p.D;
          if (col < nc) {
            const int n = T.n0 + cb + col;
            const int rowt = n / p.TT, t2 = n - rowt * p.TT, ch = t2 / p.TPW;
            const long long sl = ((long long)rowt * p.NT4 + ch) * p.TPW + (t2 - ch * p.TPW);
            dcol += (sl >> p.SBL) * 2 * bf8 + (long long)T.f * p.SB + (sl & (p.SB - 1));
          }
          for (int r = 0; r < nr; ++r) {
            const long long ro = __shfl_sync(0xffffffffu, rowoff, r);
            if (col < nc) __stcg(dcol + ro, tb[r * 33 + lane]);
          }
        }
      }
      if (p.mode == 0 && active) {
        // transpose 32 columns at a time through this warp's own 32×33 buffer (the stages
        // already hold the next tile's operands), so every store writes 128 contiguous
        // bytes of one D row
        float* tb = reinterpret_cast<float*>(smem_raw + kTcStages * kTcStageBytes) + (warp - 2) * 32 * 33;
        const int nc = min(128, T.ncols - cb);
        float* dbase = p.D + (long long)T.f * p.strideD + (long long)(T.m0 + 32 * q) * p.ldd + T.n0 + cb;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 32; ++j) tb[lane * 33 + j] = acc[32 * c + j];
          __syncwarp();
          const int col = 32 * c + lane;
          if (col < nc) {
            for (int r = 0; r < 32; ++r) {
              if (32 * q + r >= T.mrows) break;
              __stcg(dbase + (long long)r * p.ldd + col, tb[r * 33 + lane]);
            }
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

}  // namespace oaa

#ifdef OAA_DEFINE_AUX_KERNELS
namespace oaa {
// A operand of the bin GEMM, the real-ified kernel spectra, pre-split and blocked:
//   rows m < Co: (Wr at column i, −Wi at column Cip + i); rows Co + m: (Wi, Wr),
// Cip = Ci rounded up to 4 (the column layout of oaa_tile_spectra_kernel), with
// W_{o,i}[f] = DFT_P(w_{o,i})[f1][f2] / P² (fwd: o = k, i = c) or of flip180(w_{k,c})
// with o = c, i = k (bwd_data).  All other columns are zeroed by the caller.  One thread
// per (f, o, i), twiddles from a per-block fp64 table.
// P: transform size (2n − 1, or b + n − 1 for blocks b ≠ n, R18); H = (P + 1) / 2 rows
__global__ void oaa_realified_spectrum_kernel(const float* __restrict__ w, float* __restrict__ Ag, int K, int C,
                                              int n, int P, int flip_bwd, int Kc, int RTA) {
  const int H = (P + 1) / 2, F = H * P;
  const int Co = flip_bwd ? C : K, Ci = flip_bwd ? K : C, Cip = (Ci + 3) & ~3;
  __shared__ double tc[16], ts[16];
  if (threadIdx.x < P) sincospi(2.0 * (double)threadIdx.x / (double)P, &ts[threadIdx.x], &tc[threadIdx.x]);
  __syncthreads();
  const long long total = (long long)F * Co * Ci;
  const double inv = 1.0 / ((double)P * (double)P);
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    // consecutive threads take consecutive c (the fastest index of w): i for fwd (i = c),
    // o for bwd_data (o = c) -- the weight reads of a warp then stay within a few lines
    const long long kc = t % ((long long)Ci * Co);
    const int i = flip_bwd ? (int)(kc / Co) : (int)(kc % Ci);
    const int o = flip_bwd ? (int)(kc % Co) : (int)(kc / Ci);
    const int f = (int)(t / ((long long)Ci * Co));
    const int f1 = f / P, f2 = f - (f / P) * P;
    const int k = flip_bwd ? i : o, c = flip_bwd ? o : i;
    const float* wk = w + ((size_t)k * C + c) * n * n;
    double sr = 0.0, si = 0.0;
    int m1 = 0;  // (f1·p1 + f2·p2) mod P kept incrementally
    for (int p1 = 0; p1 < n; ++p1) {
      int mm = m1;
      for (int p2 = 0; p2 < n; ++p2) {
        const float v = flip_bwd ? wk[(n - 1 - p1) * n + (n - 1 - p2)] : wk[p1 * n + p2];
        sr += (double)v * tc[mm];
        si -= (double)v * ts[mm];
        mm += f2;
        if (mm >= P) mm -= P;
      }
      m1 += f1;
      if (m1 >= P) m1 -= P;
    }
    const float re = (float)(sr * inv), im = (float)(si * inv);
    tc_put_split(Ag, f, Kc, RTA, o, i, re);
    tc_put_split(Ag, f, Kc, RTA, o, Cip + i, -im);
    tc_put_split(Ag, f, Kc, RTA, Co + o, i, im);
    tc_put_split(Ag, f, Kc, RTA, Co + o, Cip + i, re);
  }
}

// Row-major X[F][rows][Kd] → pre-split blocked layout (debug entry point only).  Padding
// rows and columns are written as zeros.
__global__ void oaa_tc_pack_kernel(const float* __restrict__ X, float* __restrict__ Op, int F, int rows, int Kd,
                                   int Kc, int RT) {
  const long long total = (long long)F * RT * 128 * Kc * 32;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(t % (Kc * 32));
    const int r = (int)((t / (Kc * 32)) % (RT * 128));
    const int f = (int)(t / ((long long)Kc * 32 * RT * 128));
    const float v = (r < rows && k < Kd) ? X[((size_t)f * rows + r) * Kd + k] : 0.f;
    tc_put(Op, f, Kc, RT, r, k, v);
  }
}
}  // namespace oaa
#endif
