// oaa_kernels.cuh -- the fused sm_100a kernels of the OaA convolution layer.
//
// Notation: input blocks are n×n, transforms are P×P with
// P = 2n−1, the half spectrum keeps rows f1 ∈ [0,H), H = n, and all
// columns f2 ∈ [0,P).  A "work item" is one tile row (b, t1) of one image.
//
//  * oaa_engine_kernel<n, CR, S1>: forward and bwd_data
//    -- tile, pad, 2-D DFT, per-bin channel contraction, inverse DFT, overlap-add, crop --
//    in ONE pass.  Stage A lanes own (tile t2, spectrum row f1); stage B lanes own one
//    output column.  Horizontal overlap (n−1 columns) is resolved inside stage B by
//    summing the two contributing block columns BEFORE the last inverse transform
//    (linearity); vertical overlap (n−1 rows) is a read-modify-write of the previous
//    tile row's partial rows, ordered by a per-item release/acquire flag.
//      S1 (input-stationary): the input spectra of ≤ CR channels live in registers and
//         every output channel is contracted + inverse-transformed in turn.
//      S2 (output-stationary): ≤ CR output-channel accumulators live in registers and
//         every input channel is transformed + contracted into them.
//  * oaa_bwd_filter_kernel<n, CR>: weight gradient: per dy block s the
//    (2n−1)² x-window spectrum Ξ̂ and the block spectrum Ĝ, dŴ += conj(Ĝ)·Ξ̂, lanes own
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

constexpr int kMaxThreads = 256;  // CTA size cap: max(T·H, Ro) ≤ 256 ⇒ N ≲ 250

struct EngineParams {
  const float* in;      // [B][Cin][R][R]
  const float2* spec;   // [Cloop][Cinner][P][H]  (S1: loop=cout, S2: loop=cin)
  float* out;           // [B][Cout][Ro][Ro]
  int* flags;           // [B*T] progress of each work item (# output channels stored)
  int* counter;         // dynamic work-item counter
  int B, Cin, Cout, R, T, Ro, off, TS, num_items;
};

struct FilterParams {
  const float* x;       // [B][C][N][N]
  const float* dy;      // [B][K][M][M]
  float2* partial;      // [G][K][C][P][H]
  int B, C, K, N, M, off, Td, G, KG, TCH;
};

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Load one n×n block (rows r0.., cols c0..) of an R×R plane, zero outside (PAPER.md:18
// "rounded up" edge blocks are zero-filled; reading R13).
template <int NN>
__device__ __forceinline__ void load_block(const float* __restrict__ plane, int R, int r0, int c0,
                                           float (&z)[NN][NN]) {
#pragma unroll
  for (int p1 = 0; p1 < NN; ++p1) {
    const int r = r0 + p1;
    const bool rok = (r >= 0) && (r < R);
#pragma unroll
    for (int p2 = 0; p2 < NN; ++p2) {
      const int q = c0 + p2;
      z[p1][p2] = (rok && q >= 0 && q < R) ? __ldg(plane + (size_t)r * R + q) : 0.f;
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
    float a = 0.f, b = 0.f;
#pragma unroll
    for (int p1 = 0; p1 < NN; ++p1) {
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

// Stage A tail: inverse DFT along f2 of one spectrum row and store it, transposed, to
// the shared Q buffer  Q[f1][p2][t2]  (separate re / im planes).
template <int NN>
__device__ __forceinline__ void stage_a_store(float (&yr)[2 * NN - 1], float (&yi)[2 * NN - 1],
                                              float* __restrict__ Qr, float* __restrict__ Qi,
                                              int f1, int t2, int TS) {
  constexpr int P = 2 * NN - 1;
  float qr[P], qi[P];
  dft<P, +1>(yr, yi, qr, qi);
#pragma unroll
  for (int p2 = 0; p2 < P; ++p2) {
    Qr[(f1 * P + p2) * TS + t2] = qr[p2];
    Qi[(f1 * P + p2) * TS + t2] = qi[p2];
  }
}

// Stage B: one output column j.  Sums the two block columns that land on it, applies the
// Hermitian inverse along f1 (c2r), and writes the rows of this tile row:
//   rows p1 ∈ [n−1, 2n−1) are plain stores (p1 ≥ n are partial until the next tile row
//   adds its top rows), rows p1 ∈ [0, n−1) are added onto the previous tile row's partial
//   values once its flag says channel `ch` is stored.
template <int NN>
__device__ __forceinline__ void stage_b(const float* __restrict__ Qr, const float* __restrict__ Qi,
                                        int TS, int T, int j, int off, int Ro, int t1,
                                        float* __restrict__ plane, const int* prev_flag, int ch,
                                        int lane, unsigned bmask) {
  constexpr int P = 2 * NN - 1, H = NN;
  const int J = j + off;
  const int tA = J / NN, pA = J - tA * NN;
  const bool vA = tA < T;
  const bool vB = (tA >= 1) && (pA <= NN - 2);
  float zr[H], zi[H];
#pragma unroll
  for (int f1 = 0; f1 < H; ++f1) {
    float a = 0.f, b = 0.f;
    if (vA) { a = Qr[(f1 * P + pA) * TS + tA]; b = Qi[(f1 * P + pA) * TS + tA]; }
    if (vB) { a += Qr[(f1 * P + pA + NN) * TS + tA - 1]; b += Qi[(f1 * P + pA + NN) * TS + tA - 1]; }
    zr[f1] = a;
    zi[f1] = b;
  }
  float y[P];
  c2r_half<P>(zr, zi, y);
  const int I0 = t1 * NN - off;  // output row of block row p1 = 0
#pragma unroll
  for (int p1 = NN - 1; p1 < P; ++p1) {
    const int i = I0 + p1;
    if (i >= 0 && i < Ro) plane[(size_t)i * Ro + j] = y[p1];
  }
  if (NN > 1) {
    if (prev_flag == nullptr) {
#pragma unroll
      for (int p1 = 0; p1 < NN - 1; ++p1) {
        const int i = I0 + p1;
        if (i >= 0 && i < Ro) plane[(size_t)i * Ro + j] = y[p1];
      }
    } else {
      // one poll per warp; __syncwarp orders the other lanes' loads after the acquire
      if (lane == 0) {
        while (ld_acquire(prev_flag) < ch + 1) __nanosleep(64);
      }
      __syncwarp(bmask);
#pragma unroll
      for (int p1 = 0; p1 < NN - 1; ++p1) {
        const int i = I0 + p1;
        if (i >= 0 && i < Ro) {
          float* a = plane + (size_t)i * Ro + j;
          *a = __ldcg(a) + y[p1];
        }
      }
    }
  }
}

template <int NN, int CR, bool S1>
__global__ void __launch_bounds__(kMaxThreads, 1) oaa_engine_kernel(const EngineParams p) {
  constexpr int P = 2 * NN - 1, H = NN;
  extern __shared__ float smem[];
  __shared__ int s_item;
  const int TS = p.TS;
  const int qplane = H * P * TS;
  const int tid = threadIdx.x;
  const int lane = tid & 31;

  // stage A lane = (t2, f1)
  const int a_t = tid / H, a_f1 = tid - (tid / H) * H;
  const bool laneA = a_t < p.T;
  float cf[NN], sf[NN];
#pragma unroll
  for (int p1 = 0; p1 < NN; ++p1) {
    float s, c;
    sincospif(2.0f * (float)((a_f1 * p1) % P) / (float)P, &s, &c);
    cf[p1] = c;
    sf[p1] = s;
  }
  // stage B lane = output column j
  const bool laneB = tid < p.Ro;
  const unsigned bmask = __ballot_sync(0xffffffffu, laneB);

  for (;;) {
    if (tid == 0) s_item = atomicAdd(p.counter, 1);
    __syncthreads();
    const int item = s_item;
    if (item >= p.num_items) break;
    const int b = item / p.T, t1 = item - (item / p.T) * p.T;
    const int* prev_flag = (t1 > 0) ? (p.flags + item - 1) : nullptr;
    const float* in_b = p.in + (size_t)b * p.Cin * p.R * p.R;
    float* out_b = p.out + (size_t)b * p.Cout * p.Ro * p.Ro;
    int done = 0;  // output channels whose bottom rows are stored (published at barriers)

    if constexpr (S1) {
      float xr[CR][P], xi[CR][P];
      if (laneA) {
#pragma unroll
        for (int c = 0; c < CR; ++c) {
          if (c < p.Cin) {
            float z[NN][NN];
            load_block<NN>(in_b + (size_t)c * p.R * p.R, p.R, t1 * NN, a_t * NN, z);
            block_row_spectrum<NN>(z, cf, sf, xr[c], xi[c]);
          }
        }
      }
      for (int co = 0; co < p.Cout; ++co) {
        const int buf = co & 1;
        float* Qr = smem + buf * 2 * qplane;
        float* Qi = Qr + qplane;
        if (laneA) {
          float yr[P], yi[P];
#pragma unroll
          for (int f2 = 0; f2 < P; ++f2) { yr[f2] = 0.f; yi[f2] = 0.f; }
          const float2* s = p.spec + (size_t)co * p.Cin * P * H + a_f1;
#pragma unroll
          for (int c = 0; c < CR; ++c) {
            if (c < p.Cin) {
#pragma unroll
              for (int f2 = 0; f2 < P; ++f2) {
                const float2 w = __ldg(s + (c * P + f2) * H);
                yr[f2] = fmaf(w.x, xr[c][f2], yr[f2]);
                yr[f2] = fmaf(-w.y, xi[c][f2], yr[f2]);
                yi[f2] = fmaf(w.x, xi[c][f2], yi[f2]);
                yi[f2] = fmaf(w.y, xr[c][f2], yi[f2]);
              }
            }
          }
          stage_a_store<NN>(yr, yi, Qr, Qi, a_f1, a_t, TS);
        }
        __syncthreads();
        if (tid == 0 && co > 0) st_release(p.flags + item, co);
        if (laneB)
          stage_b<NN>(Qr, Qi, TS, p.T, tid, p.off, p.Ro, t1, out_b + (size_t)co * p.Ro * p.Ro,
                      prev_flag, co, lane, bmask);
      }
      done = p.Cout;
    } else {
      for (int c0 = 0; c0 < p.Cout; c0 += CR) {
        const int nc = min(CR, p.Cout - c0);
        float ar[CR][P], ai[CR][P];
#pragma unroll
        for (int cc = 0; cc < CR; ++cc)
#pragma unroll
          for (int f2 = 0; f2 < P; ++f2) { ar[cc][f2] = 0.f; ai[cc][f2] = 0.f; }
        if (laneA) {
          for (int ci = 0; ci < p.Cin; ++ci) {
            float z[NN][NN];
            load_block<NN>(in_b + (size_t)ci * p.R * p.R, p.R, t1 * NN, a_t * NN, z);
            float gr[P], gi[P];
            block_row_spectrum<NN>(z, cf, sf, gr, gi);
            const float2* s = p.spec + ((size_t)ci * p.Cout + c0) * P * H + a_f1;
#pragma unroll
            for (int cc = 0; cc < CR; ++cc) {
              if (cc < nc) {
#pragma unroll
                for (int f2 = 0; f2 < P; ++f2) {
                  const float2 w = __ldg(s + (cc * P + f2) * H);
                  ar[cc][f2] = fmaf(w.x, gr[f2], ar[cc][f2]);
                  ar[cc][f2] = fmaf(-w.y, gi[f2], ar[cc][f2]);
                  ai[cc][f2] = fmaf(w.x, gi[f2], ai[cc][f2]);
                  ai[cc][f2] = fmaf(w.y, gr[f2], ai[cc][f2]);
                }
              }
            }
          }
        }
#pragma unroll
        for (int cc = 0; cc < CR; ++cc) {
          if (cc < nc) {
            const int co = c0 + cc;
            const int buf = co & 1;
            float* Qr = smem + buf * 2 * qplane;
            float* Qi = Qr + qplane;
            if (laneA) stage_a_store<NN>(ar[cc], ai[cc], Qr, Qi, a_f1, a_t, TS);
            __syncthreads();
            if (tid == 0 && co > 0) st_release(p.flags + item, co);
            if (laneB)
              stage_b<NN>(Qr, Qi, TS, p.T, tid, p.off, p.Ro, t1, out_b + (size_t)co * p.Ro * p.Ro,
                          prev_flag, co, lane, bmask);
          }
        }
      }
      done = p.Cout;
    }
    __syncthreads();
    if (tid == 0) st_release(p.flags + item, done);
  }
}

// ------------------------------------------------------------------ bwd_filter
template <int NN, int CR>
__global__ void __launch_bounds__(kMaxThreads, 1) oaa_bwd_filter_kernel(const FilterParams p) {
  constexpr int P = 2 * NN - 1, H = NN;
  extern __shared__ float2 xs[];  // Ξ̂ chunk [TCH][CR][P][H]
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int kk = tid / H, f1 = tid - (tid / H) * H;
  const int k = blockIdx.y * p.KG + kk;
  const bool laneK = (kk < p.KG) && (k < p.K);
  float cf[NN], sf[NN];
#pragma unroll
  for (int p1 = 0; p1 < NN; ++p1) {
    float s, c;
    sincospif(2.0f * (float)((f1 * p1) % P) / (float)P, &s, &c);
    cf[p1] = c;
    sf[p1] = s;
  }
  const int items = p.B * p.Td;
  for (int c0 = 0; c0 < p.C; c0 += CR) {
    const int nc = min(CR, p.C - c0);
    float ar[CR][P], ai[CR][P];
#pragma unroll
    for (int cc = 0; cc < CR; ++cc)
#pragma unroll
      for (int f2 = 0; f2 < P; ++f2) { ar[cc][f2] = 0.f; ai[cc][f2] = 0.f; }
    for (int item = blockIdx.x; item < items; item += p.G) {
      const int b = item / p.Td, t1 = item - (item / p.Td) * p.Td;
      for (int tc0 = 0; tc0 < p.Td; tc0 += p.TCH) {
        const int ntc = min(p.TCH, p.Td - tc0);
        __syncthreads();
        // x-window spectra: tasks (tile tt, channel cc, row fr)
        const int ntask = ntc * nc * H;
        for (int task = tid; task < ntask; task += nthr) {
          const int fr = task % H;
          const int cc = (task / H) % nc;
          const int tt = task / (H * nc);
          const int t2 = tc0 + tt;
          const int r0 = t1 * NN + p.off - (NN - 1), q0 = t2 * NN + p.off - (NN - 1);
          const float* xp = p.x + ((size_t)b * p.C + c0 + cc) * p.N * p.N;
          float tcf[P], tsf[P];
#pragma unroll
          for (int p1 = 0; p1 < P; ++p1) {
            float s, c;
            sincospif(2.0f * (float)((fr * p1) % P) / (float)P, &s, &c);
            tcf[p1] = c;
            tsf[p1] = s;
          }
          float rr[P], ri[P];
#pragma unroll
          for (int p2 = 0; p2 < P; ++p2) {
            const int q = q0 + p2;
            const bool qok = q >= 0 && q < p.N;
            float a = 0.f, bb = 0.f;
#pragma unroll
            for (int p1 = 0; p1 < P; ++p1) {
              const int r = r0 + p1;
              const float v = (qok && r >= 0 && r < p.N) ? __ldg(xp + (size_t)r * p.N + q) : 0.f;
              a = fmaf(v, tcf[p1], a);
              bb = fmaf(-v, tsf[p1], bb);
            }
            rr[p2] = a;
            ri[p2] = bb;
          }
          float xr[P], xi[P];
          dft<P, -1>(rr, ri, xr, xi);
          float2* dst = xs + ((size_t)(tt * CR + cc) * P) * H + fr;
#pragma unroll
          for (int f2 = 0; f2 < P; ++f2) dst[f2 * H] = make_float2(xr[f2], xi[f2]);
        }
        __syncthreads();
        if (laneK) {
          const float* gp = p.dy + ((size_t)b * p.K + k) * p.M * p.M;
          for (int tt = 0; tt < ntc; ++tt) {
            const int t2 = tc0 + tt;
            float z[NN][NN];
            load_block<NN>(gp, p.M, t1 * NN, t2 * NN, z);
            float gr[P], gi[P];
            block_row_spectrum<NN>(z, cf, sf, gr, gi);
            const float2* src = xs + ((size_t)(tt * CR) * P) * H + f1;
#pragma unroll
            for (int cc = 0; cc < CR; ++cc) {
              if (cc < nc) {
#pragma unroll
                for (int f2 = 0; f2 < P; ++f2) {
                  const float2 X = src[(cc * P + f2) * H];
                  // conj(G)·X
                  ar[cc][f2] = fmaf(gr[f2], X.x, ar[cc][f2]);
                  ar[cc][f2] = fmaf(gi[f2], X.y, ar[cc][f2]);
                  ai[cc][f2] = fmaf(gr[f2], X.y, ai[cc][f2]);
                  ai[cc][f2] = fmaf(-gi[f2], X.x, ai[cc][f2]);
                }
              }
            }
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
// partial[G][K][C][P][H] → dw[K][C][n][n].  One CTA per (k, c).
__global__ void oaa_filter_finalize_kernel(const float2* __restrict__ partial, float* __restrict__ dw,
                                           int G, int K, int C, int n) {
  const int P = 2 * n - 1, H = n, bins = P * H;
  const int kc = blockIdx.x;
  extern __shared__ double2 S[];  // [P][H]
  for (int t = threadIdx.x; t < bins; t += blockDim.x) {
    double sr = 0.0, si = 0.0;
    for (int g = 0; g < G; ++g) {
      const float2 v = partial[((size_t)g * K * C + kc) * bins + t];
      sr += (double)v.x;
      si += (double)v.y;
    }
    S[t] = make_double2(sr, si);
  }
  __syncthreads();
  const double inv = 1.0 / ((double)P * (double)P);
  for (int t = threadIdx.x; t < n * n; t += blockDim.x) {
    const int u = t / n, v = t - (t / n) * n;
    const int l1 = n - 1 - u, l2 = n - 1 - v;
    double acc = 0.0;
    for (int f1 = 0; f1 < H; ++f1) {
      const double wgt = (f1 == 0) ? 1.0 : 2.0;
      for (int f2 = 0; f2 < P; ++f2) {
        const int m = (f1 * l1 + f2 * l2) % P;
        double s, c;
        sincospi(2.0 * (double)m / (double)P, &s, &c);
        const double2 z = S[f2 * H + f1];
        acc += wgt * (z.x * c - z.y * s);
      }
    }
    dw[(size_t)kc * n * n + t] = (float)(acc * inv);
  }
}

// spec[((a·Binner + bb)·P + f2)·H + f1] = DFT_P(w_kc or flip180(w_kc))[f1][f2] / P²,
// (k, c) = loop_is_k ? (a, bb) : (bb, a).
__global__ void oaa_spectrum_kernel(const float* __restrict__ w, float2* __restrict__ spec, int K,
                                    int C, int n, int flip, int loop_is_k) {
  const int P = 2 * n - 1, H = n;
  const long total = (long)K * C * P * H;
  for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < total;
       t += (long)gridDim.x * blockDim.x) {
    const int f1 = (int)(t % H);
    const int f2 = (int)((t / H) % P);
    const long ab = t / ((long)H * P);
    int k, c;
    if (loop_is_k) { k = (int)(ab / C); c = (int)(ab % C); }
    else { c = (int)(ab / K); k = (int)(ab % K); }
    const float* wk = w + ((size_t)k * C + c) * n * n;
    double sr = 0.0, si = 0.0;
    for (int p1 = 0; p1 < n; ++p1)
      for (int p2 = 0; p2 < n; ++p2) {
        const float v = flip ? wk[(n - 1 - p1) * n + (n - 1 - p2)] : wk[p1 * n + p2];
        const int m = (f1 * p1 + f2 * p2) % P;
        double s, cc;
        sincospi(2.0 * (double)m / (double)P, &s, &cc);
        sr += (double)v * cc;
        si -= (double)v * s;
      }
    const double inv = 1.0 / ((double)P * (double)P);
    spec[t] = make_float2((float)(sr * inv), (float)(si * inv));
  }
}

#endif  // OAA_DEFINE_AUX_KERNELS

}  // namespace oaa
