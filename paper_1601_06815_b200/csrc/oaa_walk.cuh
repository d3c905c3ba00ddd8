// oaa_walk.cuh -- the "walker" engine: contraction + inverse DFT + overlap-add of one
// output channel per warp, walking the tile rows of an image top to bottom.
//
// PAPER.md:18 (§2, Fig. 1): the blocks' inverse transforms "are then added with an
// overlap of n−1" to rebuild the linear convolution.  In the fused engines of
// oaa_kernels.cuh one CTA owns one tile row, so the vertical overlap (n−1 rows shared
// with the next tile row) crosses CTAs and needs progress flags, fences and a
// read-modify-write through L2.  Here one warp owns one (image, output channel) plane and
// produces its tile rows in order, so the vertical overlap never leaves the SM: the n−1
// bottom rows of tile row t1 wait in a per-warp carry buffer and are added to the top
// rows of tile row t1+1.  Every output element is written exactly once, with a plain
// streaming store, and no warp ever waits for another.
//
// A tile row is processed in chunks of TPW = ⌊32/H⌋ tiles (one warp: lanes (tt, f1)):
//   stage A  lane (tt, f1): Ŷ row f1 of tile tt = Σ_c Ŵ_c[f1,:]·X̂_c[f1,:]  (PAPER.md:15,
//            the K·C frequency-domain products summed over c; Ŵ lives in registers),
//            inverse DFT along f2 → Q[f1][p2] in the warp's shared Q ring;
//   stage B  lane = output column J of the chunk: the two block columns that land on J
//            (tile J/b at p2 = J mod b, tile J/b − 1 at p2 + b; blocks of b = n, or of
//            b = 16 − n, WalkGeo) are summed BEFORE the last transform (linearity -- the
//            horizontal overlap-add), Hermitian c2r along f1 gives the column's
//            P = b + n − 1 rows; rows [0, n−1) add the carry, rows [0, b) are final and
//            stored, rows [b, b + n − 1) become the carry.
// The forward spectra X̂ of the input blocks (one per (image, channel, block), computed
// once by oaa_xspec_kernel) stream through a ring of shared-memory chunk slots filled by
// bulk copies (TMA engine); the last warp to release a slot issues the copy that refills
// it, so there is no producer warp and no CTA barrier in the steady state.
#pragma once
#include <cuda.h>  // CUtensorMap (the tensor map itself is encoded on the host, oaa_abi.cu)
#include <cuda_runtime.h>
#include <stdint.h>

#include "dft.cuh"
#include "oaa_kernels.cuh"

namespace oaa {

// NN = kernel size n, BB = block size b (the paper's OaA has b = n; the walker
// also runs b = 16 − n for 3 ≤ n ≤ 7, SURVEY.md §8(f) NEXT-4 "block size b ≠ n"): P = b + n − 1
// is the smallest exact transform size (linear convolution of a b×b block with an n×n
// kernel), odd in both cases, so H = P2 = (P + 1) / 2 half-spectrum rows / f2 pairs.
template <int NN, int BB = NN>
struct WalkGeo {
  static constexpr int P = BB + NN - 1, H = (P + 1) / 2, P2 = (P + 1) / 2;  // f2 pairs (the last one half zero)
  static constexpr int TPW = 32 / H;                     // tiles per chunk
  static constexpr int CW = TPW * BB;                    // output columns per chunk (stage B: ⌈CW/32⌉ rounds)
  static constexpr int RS4 = P2 | 1;                     // float4 per spectrum row (odd: LDS.128 conflict free)
  static constexpr int CH4 = TPW * H * RS4;              // float4 per channel in a chunk
  static constexpr int QT = H * P;                       // float2 per tile in Q
  static constexpr int QS = 2 * TPW;                     // Q ring slots (tiles)
  static constexpr int QSZ = ((QS + 1) * QT + 1) & ~1;   // + one always-zero tile; even (16-byte multiple)
};

// Chunked spectrum layout (X̂ for fwd, Ξ̂ for bwd_filter): S[b][t1][i][c][lane][RS4]
// float4, lane = tt·H + f1, float4 q = (Re f, Im f, Re f+1, Im f+1) for f = 2q (f2 = P is
// zero).  Tiles past the last real tile (padding to NCH·TPW) are zero.
//   WIN = false: the zero-padded n×n input block of tile (t1, t2), pruned DFT;
//   WIN = true : the (2n−1)² x-window at (t1·n + org, t2·n + org) correlated with the dy
//                block in the weight gradient, full DFT.
struct XSpecParams {
  // TMA tensor map of `in` viewed as [B·Cin][R][R] (3-D, dim 0 = columns), box
  // {SW, rows, Cin}, out-of-bounds elements zero-filled: one cp.async.bulk.tensor per CTA
  // stages the zero-padded rows of all channels (the block tiler/padder of PAPER.md:18);
  // tma == 0 (R not a multiple of 4, SW > 256): per-element cp.async with zero fill.
  CUtensorMap tmap;
  const float* in;  // [B][Cin][R][R]
  float4* S;        // chunked spectra
  int Cin, R, T, NCH, SW;  // T tile rows (and columns), SW = staged row width
  int org;                 // window origin offset (WIN only)
  int tma;
};

// One CTA per (image, tile row): the rows of every channel are staged (zero padded),
// then each task (chunk i, channel c, lane) computes its block-row spectrum.
// Shared memory of oaa_xspec_kernel (256 threads): the staged input rows, then one output
// tile of CH4 float4 per warp (128-byte aligned) for the bulk stores.
__host__ __device__ inline size_t xspec_rows_floats(int Cin, int rows, int SW) {
  return ((size_t)Cin * rows * SW + 31) & ~(size_t)31;
}
inline size_t xspec_smem_bytes(int Cin, int rows, int SW, int CH4) {
  return sizeof(float) * xspec_rows_floats(Cin, rows, SW) + 8 * 16 * (size_t)CH4;
}

// BB: block size of the forward blocks (WIN = false); the x-windows (WIN) keep b = n.
template <int NN, bool WIN, int BB = NN>
__global__ void __launch_bounds__(256) oaa_xspec_kernel(const __grid_constant__ XSpecParams p) {
  static_assert(!WIN || BB == NN, "x-windows are for blocks of the kernel's size");
  using G = WalkGeo<NN, BB>;
  constexpr int P = G::P, H = G::H, RS4 = G::RS4;
  constexpr int ROWS = WIN ? P : BB;
  extern __shared__ __align__(128) float rows_s[];  // [Cin][ROWS][SW] | per-warp output tile
  __shared__ float2 tw_s[16];                        // (cos, sin)(2π m / P), m < P
  const int tid = threadIdx.x, nthr = blockDim.x;
  if (tid < P) {
    float sn, cs;
    sincospif(2.0f * (float)tid / (float)P, &sn, &cs);
    tw_s[tid] = make_float2(cs, sn);
  }
  const int item = blockIdx.x;
  const int b = item / p.T, t1 = item - (item / p.T) * p.T;
  const float* in_b = p.in + (size_t)b * p.Cin * p.R * p.R;
  const int org = WIN ? p.org : 0;
  if (p.tma) {
    __shared__ uint64_t tbar;
    if (tid == 0) {
      mbar_init(&tbar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      mbar_expect_tx(&tbar, (uint32_t)(p.SW * ROWS * p.Cin * 4));
      // box origin: column org, row t1·n + org, channel plane b·Cin (negative / past-the-end
      // coordinates are the zero padding)
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
              smem_u32(rows_s)),
          "l"(reinterpret_cast<uint64_t>(&p.tmap)), "r"(org), "r"(t1 * BB + org), "r"(b * p.Cin), "r"(smem_u32(&tbar))
          : "memory");
    }
    __syncthreads();  // (the barrier init is visible before anyone waits)
    mbar_wait(&tbar, 0);
  } else {
    const int lane = tid & 31, warp = tid >> 5, nw = nthr >> 5;
    for (int sg = warp; sg < p.Cin * ROWS; sg += nw) {
      const int c = sg / ROWS, rr = sg - (sg / ROWS) * ROWS;
      const int r = t1 * BB + org + rr;
      const bool rok = r >= 0 && r < p.R;
      const float* src = in_b + ((size_t)c * p.R + (rok ? r : 0)) * p.R;
      float* d = rows_s + (c * ROWS + rr) * p.SW;
      for (int q = lane; q < p.SW; q += 32) {
        const int col = q + org;
        const bool ok = rok && col >= 0 && col < p.R;
        cp_async4(d + q, ok ? src + col : in_b, ok);
      }
    }
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();
  }
  float4* out = p.S + (size_t)item * p.NCH * p.Cin * G::CH4;
  const int ntask = p.NCH * p.Cin * 32;
  // a thread's lane (and so its spectrum row f1) is the same for all its tasks (nthr is a
  // multiple of 32): its column twiddles e^{−2πi f1 p1 / P} come from the table once
  float tcx[WIN ? ROWS : 1], tsx[WIN ? ROWS : 1];
  if constexpr (WIN) {
    const int f1 = (tid & 31) % H;
    int m = 0;
#pragma unroll
    for (int p1 = 0; p1 < ROWS; ++p1) {
      const float2 t = tw_s[m];
      tcx[p1] = t.x;
      tsx[p1] = t.y;
      m += f1;
      if (m >= P) m -= P;
    }
  }
  for (int task = tid; task < ntask; task += nthr) {
    const int lane = task & 31, ic = task >> 5;
    const int tt0 = lane / H, f1 = lane - (lane / H) * H;
    const int tt = tt0 < G::TPW ? tt0 : 0;  // (lanes past the last tile compute a dummy row)
    const int i = ic / p.Cin, c = ic - (ic / p.Cin) * p.Cin;
    float xr[P], xi[P];
    const float* blk = rows_s + c * ROWS * p.SW;
    const int c0 = (i * G::TPW + tt) * BB;
    if constexpr (!WIN) {
      // (pruned blocks: per-task sincospif measured faster than the hoisted table values,
      // 0.143 vs 0.165 ms at the headline -- more registers live across the task loop)
      float cf[BB], sf[BB];
#pragma unroll
      for (int p1 = 0; p1 < BB; ++p1) {
        float s, co;
        sincospif(2.0f * (float)((f1 * p1) % P) / (float)P, &s, &co);
        cf[p1] = co;
        sf[p1] = s;
      }
      block_row_spectrum_smem<BB, P>(blk, p.SW, c0, cf, sf, xr, xi);
    } else {
      // column DFT of the window rows (row p1 = 0 has twiddle 1), rows read as float4
      // when the staged width keeps them 16-byte aligned (c0 = t2·n)
      float rr[P], ri[P];
#pragma unroll
      for (int p1 = 0; p1 < P; ++p1) {
        float v[P + 3];
        const float* row = blk + p1 * p.SW + c0;
        if constexpr (NN % 4 == 0) {
#pragma unroll
          for (int q = 0; q < (P + 3) / 4; ++q) {
            const float4 t = *reinterpret_cast<const float4*>(row + 4 * q);
            v[4 * q] = t.x; v[4 * q + 1] = t.y; v[4 * q + 2] = t.z; v[4 * q + 3] = t.w;
          }
        } else {
#pragma unroll
          for (int q = 0; q < P; ++q) v[q] = row[q];
        }
#pragma unroll
        for (int p2 = 0; p2 < P; ++p2) {
          if (p1 == 0) { rr[p2] = v[p2]; ri[p2] = 0.f; }
          else {
            rr[p2] = fmaf(v[p2], tcx[p1], rr[p2]);
            ri[p2] = fmaf(-v[p2], tsx[p1], ri[p2]);
          }
        }
      }
      dft<P, -1>(rr, ri, xr, xi);
    }
    // the warp's 32 rows of this task are one contiguous 32·RS4 float4 run of S: stage them
    // in the warp's smem tile and write them with one bulk copy (TMA engine)
    float4* tb = reinterpret_cast<float4*>(rows_s + xspec_rows_floats(p.Cin, ROWS, p.SW)) + (tid >> 5) * G::CH4;
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // tile free
    __syncwarp();
#pragma unroll
    for (int q = 0; q < RS4; ++q) {
      const int f = 2 * q;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (f < P) { v.x = xr[f]; v.y = xi[f]; }
      if (f + 1 < P) { v.z = xr[f + 1]; v.w = xi[f + 1]; }
      if (tt0 < G::TPW) tb[lane * RS4 + q] = v;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + (size_t)ic * G::CH4),
                   "r"(smem_u32(tb)), "r"((uint32_t)(G::CH4 * 16))
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if ((tid & 31) == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // tiles read before exit
}

struct WalkParams {
  const float4* S;     // chunked spectra (X̂: Cin channels per chunk)
  const float4* spec;  // kernel spectra [Cout][Cin][P2][H] float4 (already scaled by 1/P²)
  float* out;          // [B][Cout][Ro][Ro]
  int B, Cin, Cout, T, Ro, off, NCH;
  int KG;              // output channels (warps) per CTA
  int ngrp;            // channel groups per image = ceil(Cout / KG)
  // LOAD mode (tensor-core path): Ŷ written by the bin GEMM in its mode-2 chunk layout
  // (oaa_tc.cuh): per output channel, per (image, tile row, chunk) 2·H·P·TPW contiguous
  // floats [re/im][f1·P + f2][tile in chunk]; BTc = tiles of the batch chunk (images × T²)
  const float* D;
  int BTc, b0;
  int SBL;  // log2 of the slots per Ŷ block (oaa_tc.cuh mode 2); must equal kYSBL
  int oas;  // LOAD: the launcher picks the overlap-and-save instantiation
  int BB;   // LOAD: block size (the launcher picks the instantiation; 0 = n)
};

constexpr int kWalkRing = 4;  // spectrum chunk slots per CTA
constexpr int kYSBL = 5;      // Ŷ slot blocks of 32 (compile-time: the 30 loads of a chunk's Ŷ row
                              // then use immediate offsets, no per-load address arithmetic)

// grid = B·ngrp CTAs (image-major: the groups of one image run side by side and share
// its spectra through L2), KG warps each.
// Shared memory: ring[kWalkRing][Cin·CH4] float4 | Q[KG][QSZ] float2 |
// carry[KG][TRP/4][NCH·CW][4] floats (TRP = n−1 rounded up to 4: a column's carry rows are
// two float4, consecutive lanes' float4 contiguous).
__host__ __device__ constexpr int walk_trp(int n) { return ((n - 1) + 3) & ~3; }
// OAS = true: the overlap-and-save variant (NEXT-2 of SURVEY.md §8(f)).  S holds
// the spectra of the (2n−1)² input WINDOWS of the output blocks (oaa_xspec_kernel<n, true>,
// window origin t·n + o − (n−1)); the P-point circular convolution of a window with the
// kernel is the linear convolution on its last n rows and columns (no wrap-around), so
// stage B keeps Q column n−1+p2 and c2r rows [n−1, 2n−1) and stores them: no horizontal
// sum, no vertical carry, every output written once.
// (LOAD with n ≤ 6: no kernel spectra in registers, capped at 128 registers so that CTAs of
// 4 warps run 3 per SM -- the load walker is latency bound on its Ŷ reads; measured
// AlexNet-like fwd 0.323 → 0.304 ms, bwd_data 0.117 → 0.107 ms.  For n ≥ 7 the cap cost
// more than the occupancy gained: sharded-config fwd 4.53 → 5.29 ms per chunk.)
template <int NN, int CR, bool LOAD = false, bool OAS = false, int BB = NN>
__global__ void __launch_bounds__(256, (LOAD && BB + NN - 1 <= 11) ? 2 : 1) oaa_walk_kernel(const WalkParams p) {
  static_assert(BB == NN || !OAS, "blocks b != n: overlap-and-add only");
  using G = WalkGeo<NN, BB>;
  constexpr int P = G::P, H = G::H, P2 = G::P2, TPW = G::TPW, CW = G::CW, RS4 = G::RS4, QT = G::QT;
  constexpr int TR = NN - 1;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ uint64_t full[kWalkRing];
  __shared__ int rel[kWalkRing];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int bl = blockIdx.x / p.ngrp, grp = blockIdx.x - (blockIdx.x / p.ngrp) * p.ngrp;
  const int b = bl + (LOAD ? p.b0 : 0);
  const int co = grp * p.KG + warp;
  const int slot4 = LOAD ? 0 : p.Cin * G::CH4;  // float4 per ring slot
  float4* ring = reinterpret_cast<float4*>(smem_raw);
  float2* Qall = reinterpret_cast<float2*>(ring + kWalkRing * slot4);
  float2* Q = Qall + warp * G::QSZ;
  const int CWT = p.NCH * CW;  // carry row length
  constexpr int TRP = walk_trp(NN), TQ = TRP / 4;
  float* carry = reinterpret_cast<float*>(Qall + nw * G::QSZ) + warp * TRP * CWT;
  const int nseq = p.T * p.NCH;
  const float4* src = LOAD ? nullptr : p.S + (size_t)b * nseq * slot4;
  const uint32_t slot_bytes = (uint32_t)slot4 * 16u;

  if (tid == 0) {
    for (int s = 0; s < kWalkRing; ++s) {
      mbar_init(&full[s], 1);
      rel[s] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // zero tile of Q and the carry rows
  for (int e = lane; e < QT; e += 32) Q[G::QS * QT + e] = make_float2(0.f, 0.f);
  if constexpr (!OAS)
    for (int e = lane; e < TRP * CWT; e += 32) carry[e] = 0.f;
  __syncthreads();
  if (!LOAD && tid == 0) {
    for (int s = 0; s < kWalkRing && s < nseq; ++s) {
      mbar_expect_tx(&full[s], slot_bytes);
      bulk_g2s(ring + s * slot4, src + (size_t)s * slot4, slot_bytes, &full[s]);
    }
  }
  const bool active = co < p.Cout;  // (warp-uniform) a warp past Cout still releases slots

  // this lane's kernel spectra: Ŵ[co][c][f1 = lane mod H][f2], f2 pairs
  const int tt = lane / H, f1 = lane - (lane / H) * H;
  const bool laneA = tt < TPW;
  float4 Wr[LOAD ? 1 : CR][P2];
  if constexpr (!LOAD) {
#pragma unroll
    for (int c = 0; c < CR; ++c)
#pragma unroll
      for (int q = 0; q < P2; ++q)
        Wr[c][q] = (active && laneA && c < p.Cin) ? __ldg(p.spec + (((size_t)co * p.Cin + c) * P2 + q) * H + f1)
                                                  : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  // LOAD: this lane's Ŷ row (bins f1·P + f2) for chunk (t1, i), prefetched one chunk ahead
  float ynr[LOAD ? P : 1], yni[LOAD ? P : 1];
  // Ŷ in the layout of oaa_bin_gemm_kernel mode 2: blocks of 32 walker slots, per bin one
  // 128-byte run; the chunk's TPW slots lie in one or two blocks
  constexpr int SB = 1 << kYSBL, BF8 = SB * H * P;
  const int NT4 = (p.T + TPW - 1) / TPW;
  const size_t dplane = LOAD ? ((size_t)(p.BTc / p.T) * NT4 * TPW + SB - 1) / SB * 2 * BF8 : 0;
  const float* dlane = LOAD ? p.D + (size_t)(active ? co : 0) * dplane + f1 * P * SB : nullptr;
  auto load_y = [&](int t1, int i) {
    if constexpr (LOAD) {
      const int t2 = i * TPW + tt;
      const bool ok = active && laneA && t1 < p.T && t2 < p.T;
      const size_t sl = ((size_t)(bl * p.T + t1) * NT4 + i) * TPW + tt;
      const float* d = dlane + (ok ? (sl >> kYSBL) * 2 * BF8 + (sl & (SB - 1)) : 0);
#pragma unroll
      for (int f2 = 0; f2 < P; ++f2) {
        ynr[f2] = ok ? __ldg(d + f2 * SB) : 0.f;
        yni[f2] = ok ? __ldg(d + BF8 + f2 * SB) : 0.f;
      }
    }
  };
  if (LOAD) load_y(0, 0);
  // stage-B geometry: lane = column J = i·CW + lane (+ 32 per further round when CW > 32),
  // tile J/b = i·TPW + lq at p2 = pA
  constexpr int NRB = (CW + 31) / 32;
  const int lq = lane / BB, pA = lane - (lane / BB) * BB;
  const bool laneB = lane < CW;
  const bool hasB = pA <= NN - 2;
  const size_t plane = (size_t)p.Ro * p.Ro;
  float* outp = p.out + ((size_t)b * p.Cout + (active ? co : 0)) * plane;

  int seq = 0;
  for (int t1 = 0; t1 < p.T; ++t1) {
    const int r0 = t1 * BB - p.off;  // output row of block row 0
    unsigned rowmask = 0;            // rows p1 < b of this tile row inside [0, Ro)
#pragma unroll
    for (int p1 = 0; p1 < BB; ++p1)
      if (r0 + p1 >= 0 && r0 + p1 < p.Ro) rowmask |= 1u << p1;
    const bool rows_full = rowmask == (1u << BB) - 1u;
    for (int i = 0; i < p.NCH; ++i, ++seq) {
      const int s = seq % kWalkRing;
      if (!LOAD) mbar_wait(&full[s], (seq / kWalkRing) & 1);
      const int half = i & 1;
      // ---- stage A: contraction + inverse DFT along f2
      if constexpr (LOAD) {
        float yr[P], yi[P];
#pragma unroll
        for (int f2 = 0; f2 < P; ++f2) { yr[f2] = ynr[f2]; yi[f2] = yni[f2]; }
        if (i + 1 < p.NCH) load_y(t1, i + 1);
        else load_y(t1 + 1, 0);
        if (active && laneA) {
          float qr[P], qi[P];
          dft<P, +1>(yr, yi, qr, qi);
          float2* qd = Q + (half * TPW + tt) * QT + f1 * P;
#pragma unroll
          for (int p2 = 0; p2 < P; ++p2) qd[p2] = make_float2(qr[p2], qi[p2]);
        }
      } else {
        if (active && laneA) {
          const float4* xs = ring + s * slot4 + lane * RS4;
          float yr[P], yi[P];
#pragma unroll
          for (int c = 0; c < CR; ++c) {
            if (c < p.Cin) {
#pragma unroll
              for (int q = 0; q < P2; ++q) {
#ifdef OAA_EXP_NOXLD  // experiment builds only: X̂ from registers instead of shared memory (timing)
                const float fs = __int_as_float(0x3f800000 + (seq << 4) + c + q);
                const float4 x = make_float4(fs, -fs, fs * 0.5f, fs + 1.f);
#else
                const float4 x = xs[c * G::CH4 + q];
#endif
                const float4 w = Wr[c][q];
                const int f = 2 * q;
                if (c == 0) {
                  yr[f] = w.x * x.x;
                  yi[f] = w.x * x.y;
                } else {
                  yr[f] = fmaf(w.x, x.x, yr[f]);
                  yi[f] = fmaf(w.x, x.y, yi[f]);
                }
                yr[f] = fmaf(-w.y, x.y, yr[f]);
                yi[f] = fmaf(w.y, x.x, yi[f]);
                if (f + 1 < P) {
                  if (c == 0) {
                    yr[f + 1] = w.z * x.z;
                    yi[f + 1] = w.z * x.w;
                  } else {
                    yr[f + 1] = fmaf(w.z, x.z, yr[f + 1]);
                    yi[f + 1] = fmaf(w.z, x.w, yi[f + 1]);
                  }
                  yr[f + 1] = fmaf(-w.w, x.w, yr[f + 1]);
                  yi[f + 1] = fmaf(w.w, x.z, yi[f + 1]);
                }
              }
            }
          }
          float qr[P], qi[P];
          dft<P, +1>(yr, yi, qr, qi);
          float2* qd = Q + (half * TPW + tt) * QT + f1 * P;
#pragma unroll
          for (int p2 = 0; p2 < P; ++p2) qd[p2] = make_float2(qr[p2], qi[p2]);
        }
      }
      // release the ring slot; the last warp out refills it with chunk seq + kWalkRing
      __syncwarp();
      if (!LOAD && lane == 0) {
        __threadfence_block();
        int old;  // inc wraps to 0 after the nw-th arrival: no reset store needed
        asm volatile("atom.shared.inc.u32 %0, [%1], %2;" : "=r"(old) : "r"(smem_u32(&rel[s])), "r"(nw - 1) : "memory");
        if (old == nw - 1) {
          __threadfence_block();
          const int nx = seq + kWalkRing;
          if (nx < nseq) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(&full[s], slot_bytes);
            bulk_g2s(ring + s * slot4, src + (size_t)nx * slot4, slot_bytes, &full[s]);
          }
        }
      }
      // ---- stage B (overlap-and-save): the block's last n columns and rows, stored directly
      if constexpr (OAS) {
        if (active && laneB) {
          const int offA = (half * TPW + lq) * QT + (NN - 1) + pA;
          float zr[H], zi[H];
#pragma unroll
          for (int k = 0; k < H; ++k) {
            const float2 a = Q[offA + k * P];
            zr[k] = a.x;
            zi[k] = a.y;
          }
          float y[P];
          c2r_half<P>(zr, zi, y);
          const int j = i * CW + lane;
          if (j < p.Ro) {
            float* op = outp + (ptrdiff_t)(t1 * NN) * p.Ro + j;
#pragma unroll
            for (int r = 0; r < NN; ++r)
              if (t1 * NN + r < p.Ro) __stcs(op + (ptrdiff_t)r * p.Ro, y[NN - 1 + r]);
          }
        }
      }
      // ---- stage B: horizontal overlap-add, c2r along f1, vertical carry, stores
#pragma unroll
      for (int rb = 0; rb < NRB; ++rb) {
        const int jb = lane + 32 * rb;  // column of the chunk
        const int lqr = NRB == 1 ? lq : jb / BB, pAr = NRB == 1 ? pA : jb - (jb / BB) * BB;
        const bool hasBr = NRB == 1 ? hasB : pAr <= NN - 2;
        if (!OAS && active && (NRB == 1 ? laneB : jb < CW)) {
          const int tA = i * TPW + lqr;
          const int offA = (half * TPW + lqr) * QT + pAr;
          int offB = G::QS * QT;  // zero tile
          if (hasBr && tA >= 1) offB = (lqr > 0 ? (half * TPW + lqr - 1) : ((half ^ 1) * TPW + TPW - 1)) * QT + pAr + BB;
          float zr[H], zi[H];
#pragma unroll
          for (int k = 0; k < H; ++k) {
            const float2 a = Q[offA + k * P], bb = Q[offB + k * P];
            zr[k] = a.x + bb.x;
            zi[k] = a.y + bb.y;
          }
          float y[P];
          c2r_half<P>(zr, zi, y);
          const int J = i * CW + jb;
          const int j = J - p.off;
          float4* cr = reinterpret_cast<float4*>(carry) + J;
          float cv[TQ > 0 ? 4 * TQ : 4];
#pragma unroll
          for (int q = 0; q < TQ; ++q) {
            const float4 t = cr[q * CWT];
            cv[4 * q] = t.x; cv[4 * q + 1] = t.y; cv[4 * q + 2] = t.z; cv[4 * q + 3] = t.w;
          }
          const bool colok = j >= 0 && j < p.Ro;
          if (rows_full) {
            if (colok) {
              char* op = reinterpret_cast<char*>(outp + ((ptrdiff_t)r0 * p.Ro + j));
              const ptrdiff_t rbytes = (ptrdiff_t)p.Ro * (ptrdiff_t)sizeof(float);
#pragma unroll
              for (int p1 = 0; p1 < BB; ++p1) {
                float v = y[p1];
                if (p1 < TR) v += cv[p1];
                __stcs(reinterpret_cast<float*>(op), v);
                op += rbytes;
              }
            }
          } else {
            float* op = outp + (ptrdiff_t)r0 * p.Ro + j;
#pragma unroll
            for (int p1 = 0; p1 < BB; ++p1) {
              float v = y[p1];
              if (p1 < TR) v += cv[p1];
              if (colok && ((rowmask >> p1) & 1u)) __stcs(op + (ptrdiff_t)p1 * p.Ro, v);
            }
          }
#pragma unroll
          for (int q = 0; q < TQ; ++q) {
            float t[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) t[r] = (4 * q + r < TR) ? y[BB + 4 * q + r] : 0.f;
            cr[q * CWT] = make_float4(t[0], t[1], t[2], t[3]);
          }
        }
      }
      __syncwarp();
    }
  }
  // flush: the carry holds the last tile row's bottom rows (final)
  if (!OAS && active) {
    const int r0 = p.T * BB - p.off;
    for (int J = lane; J < p.NCH * CW; J += 32) {
      const int j = J - p.off;
      if (j < 0 || j >= p.Ro) continue;
#pragma unroll
      for (int p1 = 0; p1 < TR; ++p1) {
        const int r = r0 + p1;
        if (r >= 0 && r < p.Ro) __stcs(outp + (ptrdiff_t)r * p.Ro + j, carry[((p1 >> 2) * CWT + J) * 4 + (p1 & 3)]);
      }
    }
  }
}

}  // namespace oaa
