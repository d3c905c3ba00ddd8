// oaa_launch.cuh -- per-kernel-size launch templates.  Each oaa_inst_n<k>.cu explicitly
// instantiates them for one kernel size n so the 8 sizes compile in parallel.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "oaa_kernels.cuh"
#include "oaa_walk.cuh"
#include "oaa_bwdd.cuh"
#include "oaa_bwdf.cuh"

namespace oaa_host {
// the walker's larger block for 3 ≤ n ≤ 7: b = 16 − n, i.e. P = b + n − 1 = 15 (the n = 8 grid)
constexpr int walk_block_big(int n) { return (n >= 3 && n <= 7) ? 16 - n : n; }

extern std::atomic<uint64_t> g_launches;

// Per-kernel timing for the roofline report (oaa_profile_collect_kernels): when profiling
// is enabled, a KTimer records CUDA events on the launching stream around one launch.
enum KernelId : int {
  KID_SPECTRUM = 0,   // kernel spectra Ŵ (a1)
  KID_XSPEC,          // fwd block spectra X̂ (a2 + a3)
  KID_WALK,           // fwd walker: contraction + inverse DFT + overlap-add (a4-a6)
  KID_BWDD,           // bwd_data (a7)
  KID_XSPEC_WIN,      // bwd_filter x-window spectra Ξ̂ (a8)
  KID_BWDF,           // bwd_filter dy-block spectra + accumulation (a8)
  KID_FINALIZE,       // bwd_filter fp64 sum + inverse DFT + lag read-out (a8)
  KID_TILE_SPECTRA,   // tensor-core path: tile spectra operand (a2 + a3)
  KID_BIN_GEMM,       // tensor-core path: per-bin 3×TF32 contraction (a4)
  KID_WALK_LOAD,      // tensor-core path: inverse DFT + overlap-add of Ŷ (a5 + a6)
  KID_FILTER_SPECTRA, // tensor-core path: bwd_filter operand spectra (a8)
  KID_ENGINE,         // first-generation flag engine (shapes outside the other kernels)
  KID_AUX,            // memsets, zero tails, packing
  KID_WALK_OAS,       // overlap-and-save forward: contraction + inverse DFT + crop (NEXT-2)
  KID_BWD_FUSED,      // fused backward (NEXT-1): bwd_filter + bwd_data bodies in one launch
  KID_COUNT
};
struct KTimer {
  int kid;
  cudaStream_t s;
  void* a;
  KTimer(int kid_, cudaStream_t s_);
  ~KTimer();
};

struct EnginePlan {
  int R, Ro, off, T, Cin, Cout, TS, BW, nthreads, ncomp, CR, CIG;
  bool S1;
  bool LY;  // tensor-core path: the engine loads Ŷ computed by the bin GEMM
  size_t smem;
};

struct FilterPlan {
  int Td, KG, nkg, G, TCH, CR, nthreads, XW, DW;
  size_t smem;
};

template <int NN, int CR, bool S1>
cudaError_t launch_engine_t(const oaa::EngineParams& p, const EnginePlan& e, cudaStream_t s) {
  auto k = oaa::oaa_engine_kernel<NN, CR, S1>;
  cudaError_t err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)e.smem);
  if (err != cudaSuccess) return err;
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, e.nthreads, e.smem);
  per_sm = std::max(1, per_sm);
  const int grid = std::max(1, std::min(p.num_items, sms * per_sm));
  {
    KTimer kt(KID_ENGINE, s);
    k<<<grid, e.nthreads, e.smem, s>>>(p);
  }
  g_launches++;
  return cudaGetLastError();
}

// S1 engine with TMEM-resident input spectra: occupancy is also bounded by tensor
// memory (512 columns per SM).
template <int NN, int CR, bool LY>
cudaError_t launch_engine_s1t_t(const oaa::EngineParams& p, const EnginePlan& e, cudaStream_t s) {
  auto k = oaa::oaa_engine_s1t_kernel<NN, CR, LY>;
  cudaError_t err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)e.smem);
  if (err != cudaSuccess) return err;
  err = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (err != cudaSuccess) return err;
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, e.nthreads, e.smem);
  // (the occupancy query under-reports here; over-subscribing a persistent grid is
  // harmless: surplus CTAs find no work item and exit)
  per_sm = std::max(1, std::max(per_sm, 2));
  per_sm = std::min(per_sm, 512 / oaa::s1t_alloc_cols(NN, LY ? 0 : CR));
  const int grid = std::max(1, std::min(p.num_items, sms * per_sm));
  {
    KTimer kt(KID_ENGINE, s);
    k<<<grid, e.nthreads, e.smem, s>>>(p);
  }
  g_launches++;
  return cudaGetLastError();
}

template <int NN>
cudaError_t launch_engine_n(const oaa::EngineParams& p, const EnginePlan& e, cudaStream_t s) {
  if (e.LY) return cudaErrorInvalidValue;  // Ŷ from the bin GEMM goes through the walker (load mode)
  if (e.S1) {
    switch (e.CR) {
      case 1: return launch_engine_s1t_t<NN, 1, false>(p, e, s);
      case 2: return launch_engine_s1t_t<NN, 2, false>(p, e, s);
      case 3: return launch_engine_s1t_t<NN, 3, false>(p, e, s);
      default: return launch_engine_s1t_t<NN, 4, false>(p, e, s);
    }
  } else {
    switch (e.CR) {
      case 1: return launch_engine_t<NN, 1, false>(p, e, s);
      case 2: return launch_engine_t<NN, 2, false>(p, e, s);
      case 3: return launch_engine_t<NN, 3, false>(p, e, s);
      default: return launch_engine_t<NN, 4, false>(p, e, s);
    }
  }
}

template <int NN, int CR>
cudaError_t launch_filter_t(const oaa::FilterParams& p, const FilterPlan& f, cudaStream_t s) {
  auto k = oaa::oaa_bwd_filter_kernel<NN, CR>;
  cudaError_t err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)f.smem);
  if (err != cudaSuccess) return err;
  dim3 grid(f.G, f.nkg);
  {
    KTimer kt(KID_BWDF, s);
    k<<<grid, f.nthreads, f.smem, s>>>(p);
  }
  g_launches++;
  return cudaGetLastError();
}

template <int NN>
cudaError_t launch_filter_n(const oaa::FilterParams& p, const FilterPlan& f, cudaStream_t s) {
  switch (f.CR) {
    case 1: return launch_filter_t<NN, 1>(p, f, s);
    case 2: return launch_filter_t<NN, 2>(p, f, s);
    case 3: return launch_filter_t<NN, 3>(p, f, s);
    default: return launch_filter_t<NN, 4>(p, f, s);
  }
}

template <int NN>
cudaError_t launch_tile_spectra_n(const oaa::TileSpecParams& p, size_t smem, cudaStream_t s) {
  const bool win = p.win != 0;
  auto k = win ? oaa::oaa_tile_spectra_kernel<NN, true> : oaa::oaa_tile_spectra_kernel<NN, false>;
  if constexpr (walk_block_big(NN) != NN)
    if (!win && p.BB == walk_block_big(NN)) k = oaa::oaa_tile_spectra_kernel<NN, false, walk_block_big(NN)>;
  cudaError_t err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  {
    KTimer kt(KID_TILE_SPECTRA, s);
    const int cg = win ? 4 : 16;
    k<<<dim3(p.bc * p.T, (((p.Cin + 3) & ~3) + cg - 1) / cg), 128, smem, s>>>(p);
  }
  g_launches++;
  return cudaGetLastError();
}

template <int NN>
cudaError_t launch_filter_spectra_n(const oaa::FiltSpecParams& p, bool xwin, int items, size_t smem, cudaStream_t s) {
  auto k = xwin ? oaa::oaa_filter_spectra_kernel<NN, true> : oaa::oaa_filter_spectra_kernel<NN, false>;
  if constexpr (walk_block_big(NN) != NN)
    if (p.BB == walk_block_big(NN))
      k = xwin ? oaa::oaa_filter_spectra_kernel<NN, true, walk_block_big(NN)>
               : oaa::oaa_filter_spectra_kernel<NN, false, walk_block_big(NN)>;
  cudaError_t err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  // persistent over items: about two waves of resident CTAs, each walking items with its next
  // band prefetched
  const int groups = (p.nch + oaa::kFsCG - 1) / oaa::kFsCG;
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 32 * oaa::kFsCG, smem);
  const int gx = std::max(1, std::min(items, 2 * std::max(1, per_sm) * sms / groups));
  oaa::FiltSpecParams q = p;
  q.nitems = items;
  {
    KTimer kt(KID_FILTER_SPECTRA, s);
    k<<<dim3(gx, groups), 32 * oaa::kFsCG, smem, s>>>(q);
  }
  g_launches++;
  return cudaGetLastError();
}

// Walker forward (small Cin): block spectra X̂ of the input, then the walker.
struct WalkPlan {
  int KG, ngrp, NCH, SW;
  int BB;  // block size b: n, or walk_block_big(n) (oaa_walk.cuh WalkGeo)
  size_t xspec_smem, walk_smem;
};

template <int NN, int BB>
cudaError_t launch_walk_nb(const oaa::XSpecParams& xp, const oaa::WalkParams& wp, const WalkPlan& w, int cr,
                           cudaStream_t s) {
  {
    auto k = oaa::oaa_xspec_kernel<NN, false, BB>;
    cudaError_t err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)w.xspec_smem);
    if (err != cudaSuccess) return err;
    {
      KTimer kt(KID_XSPEC, s);
      k<<<wp.B * wp.T, 256, w.xspec_smem, s>>>(xp);
    }
    g_launches++;
    if ((err = cudaGetLastError()) != cudaSuccess) return err;
  }
  auto k = cr <= 1 ? oaa::oaa_walk_kernel<NN, 1, false, false, BB> : cr == 2 ? oaa::oaa_walk_kernel<NN, 2, false, false, BB>
         : cr == 3 ? oaa::oaa_walk_kernel<NN, 3, false, false, BB> : oaa::oaa_walk_kernel<NN, 4, false, false, BB>;
  cudaError_t err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)w.walk_smem);
  if (err != cudaSuccess) return err;
  {
    KTimer kt(KID_WALK, s);
    k<<<wp.B * w.ngrp, 32 * w.KG, w.walk_smem, s>>>(wp);
  }
  g_launches++;
  return cudaGetLastError();
}
template <int NN>
cudaError_t launch_walk_n(const oaa::XSpecParams& xp, const oaa::WalkParams& wp, const WalkPlan& w, int cr,
                          cudaStream_t s) {
  if constexpr (walk_block_big(NN) != NN)
    if (w.BB != NN) return launch_walk_nb<NN, walk_block_big(NN)>(xp, wp, w, cr, s);
  return launch_walk_nb<NN, NN>(xp, wp, w, cr, s);
}

// Overlap-and-save forward (NEXT-2): (2n−1)² input-window spectra, then the walker in OAS mode.
template <int NN>
cudaError_t launch_walk_oas_n(const oaa::XSpecParams& xp, const oaa::WalkParams& wp, size_t xspec_smem,
                              size_t walk_smem, int cr, cudaStream_t s) {
  {
    auto k = oaa::oaa_xspec_kernel<NN, true>;
    cudaError_t err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)xspec_smem);
    if (err != cudaSuccess) return err;
    {
      KTimer kt(KID_XSPEC_WIN, s);
      k<<<wp.B * wp.T, 256, xspec_smem, s>>>(xp);
    }
    g_launches++;
    if ((err = cudaGetLastError()) != cudaSuccess) return err;
  }
  auto k = cr <= 1 ? oaa::oaa_walk_kernel<NN, 1, false, true> : cr == 2 ? oaa::oaa_walk_kernel<NN, 2, false, true>
         : cr == 3 ? oaa::oaa_walk_kernel<NN, 3, false, true> : oaa::oaa_walk_kernel<NN, 4, false, true>;
  cudaError_t err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)walk_smem);
  if (err != cudaSuccess) return err;
  {
    KTimer kt(KID_WALK_OAS, s);
    k<<<wp.B * wp.ngrp, 32 * wp.KG, walk_smem, s>>>(wp);
  }
  g_launches++;
  return cudaGetLastError();
}

template <int NN, int BB>
cudaError_t launch_bwdd_nb(const oaa::BwdDParams& p, int cr, size_t smem, cudaStream_t s) {
  const bool tm = smem <= 110 * 1024;  // TMEM accumulators whenever 2 CTAs fit an SM
  auto k = tm ? (cr <= 1 ? oaa::oaa_bwdd_kernel<NN, 1, true, BB> : cr == 2 ? oaa::oaa_bwdd_kernel<NN, 2, true, BB>
                 : cr == 3 ? oaa::oaa_bwdd_kernel<NN, 3, true, BB> : oaa::oaa_bwdd_kernel<NN, 4, true, BB>)
              : (cr <= 1 ? oaa::oaa_bwdd_kernel<NN, 1, false, BB> : cr == 2 ? oaa::oaa_bwdd_kernel<NN, 2, false, BB>
                 : cr == 3 ? oaa::oaa_bwdd_kernel<NN, 3, false, BB> : oaa::oaa_bwdd_kernel<NN, 4, false, BB>);
  cudaError_t err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  {
    KTimer kt(KID_BWDD, s);
    const int ncwt = p.RPC * p.NCW;
    k<<<(p.B * p.Td + p.RPC - 1) / p.RPC, 32 * (ncwt == 7 ? 8 : ncwt), smem, s>>>(p);
  }
  g_launches++;
  return cudaGetLastError();
}
template <int NN>
cudaError_t launch_bwdd_n(const oaa::BwdDParams& p, int cr, size_t smem, cudaStream_t s) {
  if constexpr (walk_block_big(NN) != NN)
    if (p.BB != NN) return launch_bwdd_nb<NN, walk_block_big(NN)>(p, cr, smem, s);
  return launch_bwdd_nb<NN, NN>(p, cr, smem, s);
}

template <int NN>
cudaError_t launch_bwdf_n(const oaa::XSpecParams& xp, const oaa::BwdFParams& p, size_t xsmem, size_t smem, int nkg,
                          bool tm, cudaStream_t s) {
  {
    auto k = oaa::oaa_xspec_kernel<NN, true>;
    cudaError_t err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)xsmem);
    if (err != cudaSuccess) return err;
    {
      KTimer kt(KID_XSPEC_WIN, s);
      k<<<p.B * p.Td, 256, xsmem, s>>>(xp);
    }
    g_launches++;
    if ((err = cudaGetLastError()) != cudaSuccess) return err;
  }
  auto k = tm ? (p.C <= 1 ? oaa::oaa_bwdf_kernel<NN, 1, true> : p.C == 2 ? oaa::oaa_bwdf_kernel<NN, 2, true>
                : p.C == 3 ? oaa::oaa_bwdf_kernel<NN, 3, true> : oaa::oaa_bwdf_kernel<NN, 4, true>)
              : (p.C <= 1 ? oaa::oaa_bwdf_kernel<NN, 1, false> : p.C == 2 ? oaa::oaa_bwdf_kernel<NN, 2, false>
                : p.C == 3 ? oaa::oaa_bwdf_kernel<NN, 3, false> : oaa::oaa_bwdf_kernel<NN, 4, false>);
  cudaError_t err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  {
    KTimer kt(KID_BWDF, s);
    k<<<dim3(p.G, nkg), 32 * (p.KG / (32 / NN)), smem, s>>>(p);
  }
  g_launches++;
  return cudaGetLastError();
}

// Fused backward (SIMT family): Ξ̂ x-window spectra, then both backward bodies in one launch
template <int NN>
cudaError_t launch_bwd_fused_n(const oaa::XSpecParams& xp, const oaa::BwdDParams& pd, const oaa::BwdFParams& pf,
                               size_t xsmem, size_t smem, int nf, cudaStream_t s) {
  {
    auto k = oaa::oaa_xspec_kernel<NN, true>;
    cudaError_t err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)xsmem);
    if (err != cudaSuccess) return err;
    {
      KTimer kt(KID_XSPEC_WIN, s);
      k<<<pf.B * pf.Td, 256, xsmem, s>>>(xp);
    }
    g_launches++;
    if ((err = cudaGetLastError()) != cudaSuccess) return err;
  }
  auto k = pd.C <= 1 ? oaa::oaa_bwd_fused_kernel<NN, 1> : pd.C == 2 ? oaa::oaa_bwd_fused_kernel<NN, 2>
         : pd.C == 3 ? oaa::oaa_bwd_fused_kernel<NN, 3> : oaa::oaa_bwd_fused_kernel<NN, 4>;
  if constexpr (walk_block_big(NN) != NN) {
    constexpr int BG = walk_block_big(NN);
    if (pd.BB == BG)
      k = pd.C <= 1 ? oaa::oaa_bwd_fused_kernel<NN, 1, BG> : pd.C == 2 ? oaa::oaa_bwd_fused_kernel<NN, 2, BG>
        : pd.C == 3 ? oaa::oaa_bwd_fused_kernel<NN, 3, BG> : oaa::oaa_bwd_fused_kernel<NN, 4, BG>;
  }
  cudaError_t err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  {
    KTimer kt(KID_BWD_FUSED, s);
    k<<<nf + (pd.B * pd.Td + pd.RPC - 1) / pd.RPC, 256, smem, s>>>(pd, pf, nf, pf.G);
  }
  g_launches++;
  return cudaGetLastError();
}

template <int NN>
cudaError_t launch_walk_load_n(const oaa::WalkParams& wp, size_t smem, int nimg, cudaStream_t s) {
  // (oas: overlap-and-save stage B -- the blocks' last n rows / columns, no overlap-add)
  auto k = wp.oas ? oaa::oaa_walk_kernel<NN, 1, true, true> : oaa::oaa_walk_kernel<NN, 1, true>;
  if constexpr (walk_block_big(NN) != NN)
    if (!wp.oas && wp.BB == walk_block_big(NN)) k = oaa::oaa_walk_kernel<NN, 1, true, false, walk_block_big(NN)>;
  cudaError_t err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  {
    KTimer kt(KID_WALK_LOAD, s);
    k<<<nimg * wp.ngrp, 32 * wp.KG, smem, s>>>(wp);
  }
  g_launches++;
  return cudaGetLastError();
}

#define OAA_DECLARE_N(NN)                                                                      \
  extern template cudaError_t launch_engine_n<NN>(const oaa::EngineParams&, const EnginePlan&, \
                                                  cudaStream_t);                              \
  extern template cudaError_t launch_filter_n<NN>(const oaa::FilterParams&, const FilterPlan&, \
                                                  cudaStream_t);                              \
  extern template cudaError_t launch_tile_spectra_n<NN>(const oaa::TileSpecParams&, size_t, cudaStream_t); \
  extern template cudaError_t launch_filter_spectra_n<NN>(const oaa::FiltSpecParams&, bool, int, size_t, cudaStream_t); \
  extern template cudaError_t launch_walk_n<NN>(const oaa::XSpecParams&, const oaa::WalkParams&, const WalkPlan&, int, cudaStream_t); \
  extern template cudaError_t launch_bwdd_n<NN>(const oaa::BwdDParams&, int, size_t, cudaStream_t); \
  extern template cudaError_t launch_walk_oas_n<NN>(const oaa::XSpecParams&, const oaa::WalkParams&, size_t, size_t, int, cudaStream_t); \
  extern template cudaError_t launch_walk_load_n<NN>(const oaa::WalkParams&, size_t, int, cudaStream_t); \
  extern template cudaError_t launch_bwd_fused_n<NN>(const oaa::XSpecParams&, const oaa::BwdDParams&, const oaa::BwdFParams&, size_t, size_t, int, cudaStream_t); \
  extern template cudaError_t launch_bwdf_n<NN>(const oaa::XSpecParams&, const oaa::BwdFParams&, size_t, size_t, int, bool, cudaStream_t);
#define OAA_INSTANTIATE_N(NN)                                                                 \
  template cudaError_t launch_engine_n<NN>(const oaa::EngineParams&, const EnginePlan&,       \
                                           cudaStream_t);                                     \
  template cudaError_t launch_filter_n<NN>(const oaa::FilterParams&, const FilterPlan&,       \
                                           cudaStream_t);                                     \
  template cudaError_t launch_tile_spectra_n<NN>(const oaa::TileSpecParams&, size_t, cudaStream_t); \
  template cudaError_t launch_filter_spectra_n<NN>(const oaa::FiltSpecParams&, bool, int, size_t, cudaStream_t); \
  template cudaError_t launch_walk_n<NN>(const oaa::XSpecParams&, const oaa::WalkParams&, const WalkPlan&, int, cudaStream_t); \
  template cudaError_t launch_bwdd_n<NN>(const oaa::BwdDParams&, int, size_t, cudaStream_t); \
  template cudaError_t launch_walk_oas_n<NN>(const oaa::XSpecParams&, const oaa::WalkParams&, size_t, size_t, int, cudaStream_t); \
  template cudaError_t launch_walk_load_n<NN>(const oaa::WalkParams&, size_t, int, cudaStream_t); \
  template cudaError_t launch_bwd_fused_n<NN>(const oaa::XSpecParams&, const oaa::BwdDParams&, const oaa::BwdFParams&, size_t, size_t, int, cudaStream_t); \
  template cudaError_t launch_bwdf_n<NN>(const oaa::XSpecParams&, const oaa::BwdFParams&, size_t, size_t, int, bool, cudaStream_t);

}  // namespace oaa_host
