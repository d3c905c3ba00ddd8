// oaa_abi.cu -- host side of liboaa.so: argument validation, planning, workspace layout
// and kernel launches behind the C ABI declared in include/oaa.h.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/oaa.h"
#define OAA_DEFINE_AUX_KERNELS
#include "oaa_launch.cuh"
#include "oaa_tc.cuh"

namespace oaa_host {
std::atomic<uint64_t> g_launches{0};
}  // namespace oaa_host

namespace {
using namespace oaa_host;

constexpr size_t kAlign = 256;
size_t align_up(size_t v) { return (v + kAlign - 1) / kAlign * kAlign; }
int cdiv(int a, int b) { return (a + b - 1) / b; }

// ------------------------------------------------------------------ TMA tensor maps
// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link); the
// lookup runs once (thread-safe static initialisation).
PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<PFN_cuTensorMapEncodeTiled_v12000>(nullptr);
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}
// The x-block / x-window tiler of oaa_xspec_kernel: x viewed as [B·Cin][R][R] (dim 0 =
// columns), box {SW, rows, Cin} at (org, t1·n + org, b·Cin), out-of-bounds elements
// zero-filled -- the zero padding of PAPER.md:18 done by the TMA unit.  TMA needs 16-byte
// global strides (R a multiple of 4), box dimensions ≤ 256 and a non-negative box origin
// (measured: a window origin o − (n−1) < 0, i.e. Full / Same x-windows, faults with an
// illegal instruction); otherwise the kernel stages the rows with per-element cp.async
// zero fill (tma = 0).
void set_xspec_tma(oaa::XSpecParams& xp, int B, int rows) {
  xp.tma = 0;
  const PFN_cuTensorMapEncodeTiled_v12000 enc = tmap_encoder();
  if (!enc || B < 1 || xp.org != 0 || xp.R % 4 != 0 || xp.SW % 4 != 0 || xp.SW > 256 || rows > 256 || xp.Cin > 256 ||
      (reinterpret_cast<uintptr_t>(xp.in) & 15) != 0)
    return;
  const cuuint64_t dims[3] = {(cuuint64_t)xp.R, (cuuint64_t)xp.R, (cuuint64_t)B * xp.Cin};
  const cuuint64_t strides[2] = {(cuuint64_t)xp.R * 4, (cuuint64_t)xp.R * xp.R * 4};
  const cuuint32_t box[3] = {(cuuint32_t)xp.SW, (cuuint32_t)rows, (cuuint32_t)xp.Cin};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = enc(&xp.tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(xp.in), dims, strides, box,
                         estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  xp.tma = r == CUDA_SUCCESS ? 1 : 0;
}

// Ŷ of the tensor-core path (bin GEMM mode 2, walker slot = GEMM column): D viewed as the 5-D
// tensor [o][blk][ri][f][32 slots], box {32, 1, 1, 1, 32} (one drain warp's 32 rows × 32 slots),
// 128-byte swizzle (the drain buffer's XOR layout).  Needs whole 32-row groups per ri (Cf a
// multiple of 32); otherwise the drain warps store with st.global (dtma = 0).
void set_gemm_dmap(oaa::BinGemmParams& gp, long long nblk) {
  gp.dtma = 0;
  const PFN_cuTensorMapEncodeTiled_v12000 enc = tmap_encoder();
  if (!enc || gp.mode != 2 || gp.SBL != 5 || gp.TT % gp.TPW != 0 || gp.Cf % 32 != 0 || nblk < 1 ||
      (reinterpret_cast<uintptr_t>(gp.D) & 15) != 0)
    return;
  const long long bf8 = (long long)gp.SB * gp.H * gp.P;
  const cuuint64_t dims[5] = {32, (cuuint64_t)gp.H * gp.P, 2, (cuuint64_t)nblk, (cuuint64_t)gp.Cf};
  const cuuint64_t strides[4] = {32 * 4, (cuuint64_t)bf8 * 4, (cuuint64_t)bf8 * 8, (cuuint64_t)gp.plane * 4};
  const cuuint32_t box[5] = {32, 1, 1, 1, 32};
  const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  const CUresult r = enc(&gp.dmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, gp.D, dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  gp.dtma = r == CUDA_SUCCESS ? 1 : 0;
}

// ------------------------------------------------------------------ profiling
struct ProfRec {
  int op;
  cudaEvent_t a, b;
};
std::mutex g_prof_mu;
bool g_prof_on = false;
std::vector<ProfRec> g_prof;
std::vector<cudaEvent_t> g_event_pool;

cudaEvent_t get_event() {
  if (!g_event_pool.empty()) {
    cudaEvent_t e = g_event_pool.back();
    g_event_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

// per-kernel records (KTimer, oaa_launch.cuh)
struct KRec {
  int kid;
  cudaEvent_t a, b;
};
std::vector<KRec> g_kprof;

struct ProfScope {
  int op;
  cudaStream_t s;
  cudaEvent_t a = nullptr, b = nullptr;
  bool on = false;
  ProfScope(int op_, cudaStream_t s_) : op(op_), s(s_) {
    std::lock_guard<std::mutex> g(g_prof_mu);
    on = g_prof_on;
    if (on) {
      a = get_event();
      b = get_event();
    }
  }
  void start() { if (on) cudaEventRecord(a, s); }
  void stop() {
    if (!on) return;
    cudaEventRecord(b, s);
    std::lock_guard<std::mutex> g(g_prof_mu);
    g_prof.push_back({op, a, b});
  }
};

}  // namespace

namespace oaa_host {
KTimer::KTimer(int kid_, cudaStream_t s_) : kid(kid_), s(s_), a(nullptr) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  if (!g_prof_on) return;
  cudaEvent_t e = get_event();
  cudaEventRecord(e, s);
  a = e;
}
KTimer::~KTimer() {
  if (!a) return;
  std::lock_guard<std::mutex> g(g_prof_mu);
  cudaEvent_t e = get_event();
  cudaEventRecord(e, s);
  g_kprof.push_back({kid, static_cast<cudaEvent_t>(a), e});
}
}  // namespace oaa_host

namespace {
// ---------------------------------------------------------------- geometry
struct Geo {
  int n, P, H, M, o;
};

bool make_geo(int N, int n, oaa_crop_t crop, Geo* g) {
  if (N < 1 || n < 1) return false;
  int M = oaa_conv_out_size(N, n, crop);
  if (M < 1) return false;
  g->n = n;
  g->P = 2 * n - 1;
  g->H = n;
  g->M = M;
  g->o = crop == OAA_CROP_FULL ? 0 : crop == OAA_CROP_VALID ? n - 1 : (n - 1) / 2;
  return true;
}

// register channel capacity of the engine: CR ∈ {1..4}
constexpr int kCRMax = 4;


bool plan_engine(int R, int Ro, int off, int n, int Cin, int Cout, EnginePlan* e, bool ly = false) {
  e->LY = ly;
  e->R = R;
  e->Ro = Ro;
  e->off = off;
  e->T = cdiv(R, n);
  e->Cin = Cin;
  e->Cout = Cout;
  const int laneA = e->T * n;
  const int need = std::max(laneA, Ro);
  if (need > oaa::kMaxThreads) return false;
  e->ncomp = cdiv(need, 32) * 32;
  e->nthreads = e->ncomp + 32 <= oaa::kMaxThreads ? e->ncomp + 32 : e->ncomp;  // + publisher warp
  e->TS = oaa::q_stride(n);
  e->BW = cdiv(e->T * n, 4) * 4;
  const int P = 2 * n - 1, H = n, P2 = (P + 1) / 2;
  if (Cin <= kCRMax) {
    e->S1 = true;
    e->CR = Cin;
  } else {
    e->S1 = false;
    e->CR = std::min(Cout, kCRMax);
  }
  const size_t q_b = sizeof(float2) * 2 * ((size_t)H * P * e->TS);
  if (ly) {
    // the engine only inverts Ŷ (bin GEMM output) and overlap-adds: no inputs, no spectra
    e->S1 = true;
    e->CR = 1;
    e->CIG = 1;
    e->smem = q_b;
  } else if (e->S1) {
    // S1 runs the TMEM engine (spectra and deferred rows in tensor memory, no smem ring)
    e->CIG = 1;
    e->smem = q_b + sizeof(float4) * (size_t)3 * Cin * P2 * H + sizeof(float) * (size_t)Cin * n * e->BW;
  } else {
    const size_t ring_b = sizeof(float) * (size_t)std::min(oaa::kRingDepth, Cout) * (n - 1) * oaa::kMaxThreads;
    for (e->CIG = 4; e->CIG >= 1; e->CIG /= 2) {
      e->smem = q_b + ring_b + 2 * (size_t)e->CIG * (sizeof(float4) * (size_t)e->CR * P2 * H + sizeof(float) * (size_t)n * e->BW);
      if (e->smem <= 220 * 1024) break;
    }
    if (e->CIG < 1) e->CIG = 1;
  }
  return e->smem <= 220 * 1024;
}

bool plan_filter(int B, int C, int K, int M, int n, FilterPlan* f) {
  const int H = n, P = 2 * n - 1;
  f->Td = cdiv(M, n);
  f->KG = std::max(1, oaa::kMaxThreads / H);
  f->KG = std::min(f->KG, K);
  f->nkg = cdiv(K, f->KG);
  f->nthreads = cdiv(f->KG * H, 32) * 32;
  f->TCH = std::max(1, std::min(f->Td, 32 / n));
  f->XW = cdiv(f->Td * n + n - 1, 4) * 4;
  f->DW = cdiv(f->TCH * n, 4) * 4;
  // channels per pass: as many as fit (the Ξ̂ of a whole tile row grows with Td·CR)
  for (f->CR = std::min(C, kCRMax); f->CR >= 1; --f->CR) {
    f->smem = sizeof(float) * (size_t)f->CR * P * f->XW + sizeof(float2) * (size_t)f->Td * f->CR * P * H +
              2 * sizeof(float) * (size_t)f->KG * n * f->DW + sizeof(float2) * 16;
    if (f->smem <= 220 * 1024) break;
  }
  if (f->CR < 1) f->CR = 1;
  const int items = std::max(1, B * f->Td);
  // one persistent wave: ~148 SMs on B200 (fixed so results do not depend on the device)
  f->G = std::max(1, std::min(items, 148 / f->nkg));
  return f->smem <= 220 * 1024;
}

// ---------------------------------------------------------------- dispatch
}  // namespace
namespace oaa_host {
OAA_DECLARE_N(1)
OAA_DECLARE_N(2)
OAA_DECLARE_N(3)
OAA_DECLARE_N(4)
OAA_DECLARE_N(5)
OAA_DECLARE_N(6)
OAA_DECLARE_N(7)
OAA_DECLARE_N(8)
}  // namespace oaa_host
namespace {

cudaError_t launch_engine(int n, const oaa::EngineParams& p, const EnginePlan& e, cudaStream_t s) {
  switch (n) {
    case 1: return launch_engine_n<1>(p, e, s);
    case 2: return launch_engine_n<2>(p, e, s);
    case 3: return launch_engine_n<3>(p, e, s);
    case 4: return launch_engine_n<4>(p, e, s);
    case 5: return launch_engine_n<5>(p, e, s);
    case 6: return launch_engine_n<6>(p, e, s);
    case 7: return launch_engine_n<7>(p, e, s);
    case 8: return launch_engine_n<8>(p, e, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_walk(int n, const oaa::XSpecParams& xp, const oaa::WalkParams& wp, const WalkPlan& w, int cr,
                        cudaStream_t s) {
  switch (n) {
    case 1: return launch_walk_n<1>(xp, wp, w, cr, s);
    case 2: return launch_walk_n<2>(xp, wp, w, cr, s);
    case 3: return launch_walk_n<3>(xp, wp, w, cr, s);
    case 4: return launch_walk_n<4>(xp, wp, w, cr, s);
    case 5: return launch_walk_n<5>(xp, wp, w, cr, s);
    case 6: return launch_walk_n<6>(xp, wp, w, cr, s);
    case 7: return launch_walk_n<7>(xp, wp, w, cr, s);
    case 8: return launch_walk_n<8>(xp, wp, w, cr, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_walk_load(int n, const oaa::WalkParams& wp, size_t smem, int nimg, cudaStream_t s) {
  switch (n) {
    case 1: return launch_walk_load_n<1>(wp, smem, nimg, s);
    case 2: return launch_walk_load_n<2>(wp, smem, nimg, s);
    case 3: return launch_walk_load_n<3>(wp, smem, nimg, s);
    case 4: return launch_walk_load_n<4>(wp, smem, nimg, s);
    case 5: return launch_walk_load_n<5>(wp, smem, nimg, s);
    case 6: return launch_walk_load_n<6>(wp, smem, nimg, s);
    case 7: return launch_walk_load_n<7>(wp, smem, nimg, s);
    case 8: return launch_walk_load_n<8>(wp, smem, nimg, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_bwdd(int n, const oaa::BwdDParams& p, int cr, size_t smem, cudaStream_t s) {
  switch (n) {
    case 1: return launch_bwdd_n<1>(p, cr, smem, s);
    case 2: return launch_bwdd_n<2>(p, cr, smem, s);
    case 3: return launch_bwdd_n<3>(p, cr, smem, s);
    case 4: return launch_bwdd_n<4>(p, cr, smem, s);
    case 5: return launch_bwdd_n<5>(p, cr, smem, s);
    case 6: return launch_bwdd_n<6>(p, cr, smem, s);
    case 7: return launch_bwdd_n<7>(p, cr, smem, s);
    case 8: return launch_bwdd_n<8>(p, cr, smem, s);
  }
  return cudaErrorInvalidValue;
}

struct BwdfLaunch {
  size_t xspec_smem, smem;
  int nkg;
  bool tm;
};
cudaError_t launch_bwdf(int n, const oaa::XSpecParams& xp, const oaa::BwdFParams& fp, const BwdfLaunch& f,
                        cudaStream_t s) {
  switch (n) {
    case 1: return launch_bwdf_n<1>(xp, fp, f.xspec_smem, f.smem, f.nkg, f.tm, s);
    case 2: return launch_bwdf_n<2>(xp, fp, f.xspec_smem, f.smem, f.nkg, f.tm, s);
    case 3: return launch_bwdf_n<3>(xp, fp, f.xspec_smem, f.smem, f.nkg, f.tm, s);
    case 4: return launch_bwdf_n<4>(xp, fp, f.xspec_smem, f.smem, f.nkg, f.tm, s);
    case 5: return launch_bwdf_n<5>(xp, fp, f.xspec_smem, f.smem, f.nkg, f.tm, s);
    case 6: return launch_bwdf_n<6>(xp, fp, f.xspec_smem, f.smem, f.nkg, f.tm, s);
    case 7: return launch_bwdf_n<7>(xp, fp, f.xspec_smem, f.smem, f.nkg, f.tm, s);
    case 8: return launch_bwdf_n<8>(xp, fp, f.xspec_smem, f.smem, f.nkg, f.tm, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_filter(int n, const oaa::FilterParams& p, const FilterPlan& f, cudaStream_t s) {
  switch (n) {
    case 1: return launch_filter_n<1>(p, f, s);
    case 2: return launch_filter_n<2>(p, f, s);
    case 3: return launch_filter_n<3>(p, f, s);
    case 4: return launch_filter_n<4>(p, f, s);
    case 5: return launch_filter_n<5>(p, f, s);
    case 6: return launch_filter_n<6>(p, f, s);
    case 7: return launch_filter_n<7>(p, f, s);
    case 8: return launch_filter_n<8>(p, f, s);
  }
  return cudaErrorInvalidValue;
}

bool overlaps(const void* a, size_t an, const void* b, size_t bn) {
  const char* pa = static_cast<const char*>(a);
  const char* pb = static_cast<const char*>(b);
  return pa < pb + bn && pb < pa + an;
}

// Common validation. Returns OAA_OK or an error without touching memory.
oaa_status_t validate(int B, int C, int K, int N, int n, oaa_crop_t crop, Geo* g) {
  if (B < 0 || C < 1 || K < 1 || N < 1 || n < 1) return OAA_ERR_INVALID_VALUE;
  if (crop != OAA_CROP_FULL && crop != OAA_CROP_VALID && crop != OAA_CROP_SAME)
    return OAA_ERR_INVALID_VALUE;
  if (!make_geo(N, n, crop, g)) return OAA_ERR_INVALID_VALUE;
  if (n > 8) return OAA_ERR_UNSUPPORTED;
  return OAA_OK;
}

// tensor-core path ----------------------------------------------
// Layers with many input AND output channels evaluate the per-bin contraction as a
// real-ified GEMM on the tensor cores (oaa_tc.cuh): tile spectra Xg → D = Ag·Xgᵀ → the
// walker (load mode) inverts and overlap-adds.  Xg and D hold one batch chunk at a time.
constexpr int kTcMinChannels = 16;
constexpr size_t kTcChunkBytes = size_t(1) << 33;  // Xg + D per chunk (8 GB: launches large enough to fill the GPU)

struct TcPlan {
  bool use;
  int BB, P, H;  // block size b (n, or 16 − n: DESIGN.md R18), transform size, spectrum rows
  int F, T, Kc, RTA, RTB, NB, bc, nchunks;  // K chunks of 32, row tiles of A and B, B tiles per CTA
  bool b_split;  // B (block spectra) stored pre-split: each B tile is re-read by RTA ≥ 3 M tiles
  size_t ag_b, xg_b, d_b;
};
// allow_big = false: blocks of the kernel's size (the fused backward, whose weight-gradient
// producers share the dy tiling, and overlap-and-save keep b = n)
TcPlan plan_tc(int B, int Cin, int Cout, int R, int n, bool allow_big = true) {
  TcPlan t{};
  t.use = Cin >= kTcMinChannels && Cout >= kTcMinChannels;
  if (!t.use || B < 1) return t;
  // larger blocks as the walker's (plan_walk), P = 15, for n = 6, 7 only, whose own grids P = 11,
  // 13 are primes (costly pairing codelets in the tile producer and the load walker): measured
  // B = 128 C = 32 K = 64 N = 64 n = 7 fwd 1.009 → 0.523 ms, bwd_data 0.770 → 0.592.  For n ≤ 5
  // the tensor cores make the contraction cheap and the P = 15 producer / walker cost more than
  // the bins they save (N = 56 n = 3 fwd 0.500 → 0.541; configs[3] n = 5 fwd 0.888 → 1.317).
  const int big = walk_block_big(n);
  const long long pad = (long long)cdiv(R, big) * big;
#ifdef OAA_EXP_TC_SMALLB  // experiment builds only: the tensor-core path keeps b = n
  t.BB = n;
#elif defined(OAA_EXP_TC_BIG_ALL)  // experiment builds only: larger blocks for every 3 ≤ n ≤ 7
  t.BB = (allow_big && big != n && (R >= 3 * big || (R >= 2 * big && 2 * pad * pad <= 3LL * R * R))) ? big : n;
#else
  t.BB = (allow_big && n >= 6 && big != n && (R >= 3 * big || (R >= 2 * big && 2 * pad * pad <= 3LL * R * R))) ? big : n;
#endif
  t.P = t.BB + n - 1;
  t.H = (t.P + 1) / 2;
  t.F = t.H * t.P;
  t.T = cdiv(R, t.BB);
  t.Kc = cdiv(2 * ((Cin + 3) & ~3), oaa::kTcK);
  t.RTA = cdiv(2 * Cout, oaa::kTcM);
  // measured (AlexNet-like fwd, 4 M tiles): splitting B once in HBM beats re-splitting every
  // re-read in the GEMM; with ≤ 2 M tiles the halved operand bytes win
  t.b_split = t.RTA >= 3;
  const size_t per_img = sizeof(float) * (size_t)t.F * t.T * t.T *
                         ((t.b_split ? 2 : 1) * (size_t)t.Kc * oaa::kTcK + 2 * (size_t)Cout);
  t.nchunks = (int)std::max<size_t>(1, (B * per_img + kTcChunkBytes - 1) / kTcChunkBytes);
  t.bc = cdiv(B, t.nchunks);
  t.nchunks = cdiv(B, t.bc);
  t.NB = t.bc * t.T * t.T > oaa::kTcM ? 2 : 1;
  t.RTB = cdiv(cdiv(t.bc * t.T * t.T, oaa::kTcM), t.NB) * t.NB;
  t.ag_b = sizeof(float) * (size_t)t.F * t.Kc * 2 * t.RTA * 4096;  // pre-split (hi | lo)
  t.xg_b = sizeof(float) * (size_t)t.F * t.Kc * (t.b_split ? 2 : 1) * t.RTB * 4096;
  // Ŷ in the walker layout (oaa_tc.cuh mode 2): tile rows padded to whole walker chunks
  const int TPW = 32 / t.H;
  t.d_b = sizeof(float) * (size_t)t.F * 2 * Cout * ((size_t)t.bc * t.T * (cdiv(t.T, TPW) * TPW) + 31) / 32 * 32;
  return t;
}

// walker forward (oaa_walk.cuh): small input-channel counts, forward only -------------
constexpr int kWalkMaxCin = 4;
struct WalkHostGeo {
  bool use;
  int BB, P, H, T, TPW, CW, RS4, CH4, NCH, KG, ngrp;  // BB = block size b, T = ⌈R / b⌉ tiles per side
  size_t spec_b, xs_b;
};
WalkHostGeo plan_walk(bool is_fwd, int B, int Cin, int Cout, int R, int Ro, int off, int n, const TcPlan& tc) {
  WalkHostGeo w{};
  w.use = is_fwd && !tc.use && Cin <= kWalkMaxCin;
  // block size: for 3 ≤ n ≤ 7 the blocks grow to
  // b = 16 − n, so every block uses the P = 15 grid of n = 8 (PFA 3×5 codelets, 8 spectrum rows,
  // 4 blocks per warp) and yields b² instead of n² outputs -- once the image holds ≥ 3 of them,
  // or 2 with at most 1.5× the image area in padded blocks (measured at N = 32, B = 128, C = 3,
  // K = 64: n = 3 / 5 walk 0.080 → 0.055 ms; at N = 20, n = 7, 1.8× area, 0.043 → 0.052)
  const int big = walk_block_big(n);
  const long long pad = (long long)cdiv(R, big) * big;
  w.BB = (big != n && (R >= 3 * big || (R >= 2 * big && 2 * pad * pad <= 3LL * R * R))) ? big : n;
  w.P = w.BB + n - 1;
  w.H = (w.P + 1) / 2;
  w.T = cdiv(R, w.BB);
  w.TPW = 32 / w.H;
  w.CW = w.TPW * w.BB;
  w.RS4 = w.H | 1;
  w.CH4 = w.TPW * w.H * w.RS4;
  w.NCH = cdiv(off + Ro, w.CW);
  w.KG = std::min(8, Cout);
  w.ngrp = cdiv(Cout, w.KG);
  w.spec_b = align_up(sizeof(float4) * (size_t)Cin * Cout * w.H * w.H);
  w.xs_b = align_up(sizeof(float4) * (size_t)B * w.T * w.NCH * Cin * w.CH4);
  return w;
}

// overlap-and-save forward (NEXT-2; the walker in OAS mode) -----------------------------
struct OasPlan {
  bool use;
  int Td, TPW, CW, CH4, NCH, KG, ngrp, SW;
  size_t spec_b, xs_b, xspec_smem, walk_smem;
};
OasPlan plan_oas(int B, int C, int K, int N, int n, const Geo& g) {
  OasPlan o{};
  o.use = C <= kWalkMaxCin;
  const int P = 2 * n - 1;
  o.Td = cdiv(g.M, n);
  o.TPW = 32 / n;
  o.CW = o.TPW * n;
  o.CH4 = o.TPW * n * (n | 1);
  o.NCH = cdiv(g.M, o.CW);
  o.KG = std::min(8, K);
  o.ngrp = cdiv(K, o.KG);
  o.SW = cdiv(o.NCH * o.CW + n - 1, 4) * 4;
  o.spec_b = align_up(sizeof(float4) * (size_t)C * K * n * n);
  o.xs_b = align_up(sizeof(float4) * (size_t)B * o.Td * o.NCH * C * o.CH4);
  o.xspec_smem = oaa::xspec_smem_bytes(C, P, o.SW, o.CH4);
  const int QSZ = ((2 * o.TPW + 1) * n * P + 1) & ~1;
  o.walk_smem = sizeof(float4) * (size_t)oaa::kWalkRing * C * o.CH4 + sizeof(float2) * (size_t)o.KG * QSZ;
  if (o.walk_smem > 220 * 1024 || o.xspec_smem > 220 * 1024) o.use = false;
  (void)N;
  return o;
}
cudaError_t launch_walk_oas(int n, const oaa::XSpecParams& xp, const oaa::WalkParams& wp, const OasPlan& o, int cr,
                            cudaStream_t s) {
  switch (n) {
    case 1: return launch_walk_oas_n<1>(xp, wp, o.xspec_smem, o.walk_smem, cr, s);
    case 2: return launch_walk_oas_n<2>(xp, wp, o.xspec_smem, o.walk_smem, cr, s);
    case 3: return launch_walk_oas_n<3>(xp, wp, o.xspec_smem, o.walk_smem, cr, s);
    case 4: return launch_walk_oas_n<4>(xp, wp, o.xspec_smem, o.walk_smem, cr, s);
    case 5: return launch_walk_oas_n<5>(xp, wp, o.xspec_smem, o.walk_smem, cr, s);
    case 6: return launch_walk_oas_n<6>(xp, wp, o.xspec_smem, o.walk_smem, cr, s);
    case 7: return launch_walk_oas_n<7>(xp, wp, o.xspec_smem, o.walk_smem, cr, s);
    case 8: return launch_walk_oas_n<8>(xp, wp, o.xspec_smem, o.walk_smem, cr, s);
  }
  return cudaErrorInvalidValue;
}

// bwd_data for few output channels (oaa_bwdd.cuh) ------------------------------------
struct BwddPlan {
  bool use;
  int BB, P, H, Td;  // dy block size b (as the forward walker's, plan_walk), grid, tiles per side
  int NCW, BW, RPC, WSL;
  size_t smem;
};
// allow_big = false: blocks of the kernel's size
BwddPlan plan_bwdd(bool is_fwd, int B, int Cout, int R, int n, const TcPlan& tc, bool allow_big = true) {
  BwddPlan d{};
  d.use = !is_fwd && !tc.use && Cout <= kWalkMaxCin;
  // (the larger blocks from 3 per side for n ≤ 4, from R ≥ 96 for n ≥ 5: measured at R = 58-60,
  // n = 5 / 7, the fewer, larger blocks leave too few warps per CTA, 0.155 → 0.185 ms at n = 5)
  const int big = walk_block_big(n);
  d.BB = (allow_big && big != n && R >= 3 * big && (n <= 4 || R >= 96)) ? big : n;
  d.P = d.BB + n - 1;
  d.H = (d.P + 1) / 2;
  const int TPW = 32 / d.H, CW = TPW * d.BB;
  d.Td = cdiv(R, d.BB);
  d.NCW = cdiv(d.Td, TPW);
  if (d.NCW > 8) d.use = false;  // ≤ 8 warps (256 threads)
  d.BW = d.NCW * CW;
  // narrow images: several (image, tile row) pairs per CTA so that it has 8 compute warps
  // sharing one Ŵ ring (a half-depth ring keeps two such CTAs per SM); the headline's 7
  // chunk warps keep one pair and the 16-deep ring
  // while keeping ≥ 2 CTAs per SM of work
  d.RPC = (d.NCW >= 1 && d.NCW <= 4) ? std::max(1, std::min(8 / d.NCW, B * d.Td / 296)) : 1;
  d.WSL = d.RPC > 1 ? 3 : 4;
  d.smem = oaa::bwdd_smem_bytes(n, d.BB, Cout, d.NCW, d.RPC, d.WSL);
  if (d.smem > 220 * 1024) d.use = false;
  return d;
}

// bwd_filter for few input channels (oaa_bwdf.cuh) ------------------------------------
struct BwdfPlan {
  bool use;
  int TPW, CW, CH4, NCH, Td, KPW, nkg, nwb, KG, G, SW;
  bool tm;
  size_t xs_b, part_b, xspec_smem, smem;
};
BwdfPlan plan_bwdf(int B, int C, int K, int M, int n) {
  BwdfPlan f{};
  f.use = C <= kWalkMaxCin && B > 0;
  const int H = n, P = 2 * n - 1;
  f.TPW = 32 / H;
  f.CW = f.TPW * n;
  f.CH4 = f.TPW * H * (n | 1);
  f.Td = cdiv(M, n);
  f.NCH = cdiv(f.Td, f.TPW);
  f.KPW = 32 / H;
  f.nkg = cdiv(K, oaa::kBwdfWarps * f.KPW);
  // balanced kernel groups: each CTA takes ⌈K / nkg⌉ kernels rounded up to whole warps
  f.nwb = cdiv(cdiv(K, f.nkg), f.KPW);
  f.KG = f.nwb * f.KPW;
  // TMEM accumulators for n ≥ 6 (C·P complex per lane would not fit 128 registers; measured
  // faster than registers at 1 CTA / SM); registers for n ≤ 5, where the per-block
  // TMEM ld + st of 32 columns per channel outweighs the C·P·4 FMAs it serves
#ifdef OAA_EXP_BWDF_TM_ALL  // experiment builds only: tensor-memory accumulators for every n
  f.tm = true;
#else
  f.tm = n >= 6;
#endif
  int slots = 296;
  f.G = std::max(1, std::min(B * f.Td, slots / f.nkg));
  f.SW = cdiv(f.NCH * f.CW + n - 1, 4) * 4;
  f.xs_b = align_up(sizeof(float4) * (size_t)B * f.Td * f.NCH * C * f.CH4);
  f.part_b = align_up(sizeof(float2) * (size_t)f.G * K * C * P * H);
  f.xspec_smem = oaa::xspec_smem_bytes(C, P, f.SW, f.CH4);
  f.smem = f.tm ? oaa::bwdf_smem_bytes<true>(n, C) : oaa::bwdf_smem_bytes<false>(n, C);
  if (f.smem > 220 * 1024 || f.xspec_smem > 220 * 1024) f.use = false;
  return f;
}

// workspace layouts ------------------------------------------------------------
struct EngineWs {
  size_t spec_off, flags_off, counter_off, xg_off, d_off, total;
};
EngineWs engine_ws(int B, int C, int K, int Tr, const Geo& g, const TcPlan& tc, const WalkHostGeo* wk = nullptr,
                   const BwddPlan* bd = nullptr) {
  EngineWs w{};
  w.spec_off = 0;
  if (bd && bd->use) {
    w.flags_off = w.counter_off = w.d_off = w.xg_off = 0;
    w.total = align_up(sizeof(float4) * (size_t)K * C * bd->H * bd->H);
    return w;
  }
  if (wk && wk->use) {
    w.xg_off = wk->spec_b;  // X̂ chunks
    w.flags_off = w.counter_off = w.d_off = 0;
    w.total = wk->spec_b + wk->xs_b;
    return w;
  }
  if (tc.use) {
    w.flags_off = align_up(tc.ag_b);
    w.counter_off = align_up(w.flags_off + sizeof(int) * (size_t)std::max(1, tc.bc * Tr));
    w.xg_off = align_up(w.counter_off + sizeof(int));
    w.d_off = align_up(w.xg_off + tc.xg_b);
    w.total = align_up(w.d_off + tc.d_b);
    return w;
  }
  w.flags_off = align_up(sizeof(float4) * (size_t)K * C * ((g.P + 1) / 2) * g.H);
  w.counter_off = align_up(w.flags_off + sizeof(int) * (size_t)std::max(1, B * Tr));
  w.total = align_up(w.counter_off + sizeof(int));
  return w;
}

cudaError_t launch_tile_spectra(int n, const oaa::TileSpecParams& p, size_t smem, cudaStream_t s) {
  switch (n) {
    case 1: return launch_tile_spectra_n<1>(p, smem, s);
    case 2: return launch_tile_spectra_n<2>(p, smem, s);
    case 3: return launch_tile_spectra_n<3>(p, smem, s);
    case 4: return launch_tile_spectra_n<4>(p, smem, s);
    case 5: return launch_tile_spectra_n<5>(p, smem, s);
    case 6: return launch_tile_spectra_n<6>(p, smem, s);
    case 7: return launch_tile_spectra_n<7>(p, smem, s);
    case 8: return launch_tile_spectra_n<8>(p, smem, s);
  }
  return cudaErrorInvalidValue;
}

// tensor-core weight gradient: Ĝ / Ξ̂ spectra of a batch chunk →
// split-K bin GEMM writing per-split partial dŴ → the fp64 finalize of the FFMA path.
struct TcFiltPlan {
  bool use;
  int BB, P, H;  // dy block size (n, or 16 − n for n = 6, 7 as plan_tc), grid, spectrum rows
  int F, Td, T2, RTA, RTB, NB, bc, nchunks, Kc, S, kps, G, SWg, SWx;
  size_t a_b, b_b, part_b;
};
// bc_force / bb_force (fused backward): the data path's batch chunk and dy block size
TcFiltPlan plan_tc_filter(int B, int C, int K, int N, int M, int n, int bc_force = 0, int bb_force = 0) {
  TcFiltPlan t{};
  t.use = C >= kTcMinChannels && K >= kTcMinChannels;
  if (!t.use || B < 1) return t;
  // blocks b = 16 − n on the P = 15 grid for n = 6, 7 (their own P = 11, 13 are primes; as
  // plan_tc); the fused backward passes its data path's block size (bb_force), whose Ĝ it reads
  const int big = walk_block_big(n);
  const long long pad = (long long)cdiv(M, big) * big;
#ifdef OAA_EXP_TC_SMALLB  // experiment builds only: b = n
  t.BB = n;
#else
  t.BB = (n >= 6 && big != n && (M >= 3 * big || (M >= 2 * big && 2 * pad * pad <= 3LL * M * M))) ? big : n;
#endif
  if (bb_force > 0) t.BB = bb_force;
  t.P = t.BB + n - 1;
  t.H = (t.P + 1) / 2;
  t.F = t.H * t.P;
  t.Td = cdiv(M, t.BB);
  t.T2 = t.Td * t.Td;
  t.RTA = cdiv(K, oaa::kTcM);
  t.NB = 2 * C > oaa::kTcM ? 2 : 1;
  t.RTB = cdiv(cdiv(2 * C, oaa::kTcM), t.NB) * t.NB;
  const size_t per_img = sizeof(float) * (size_t)t.F * 2 * t.T2 * 128 * (size_t)(t.RTA + t.RTB);
  t.nchunks = (int)std::max<size_t>(1, (B * per_img + kTcChunkBytes - 1) / kTcChunkBytes);
  t.bc = cdiv(B, t.nchunks);
  if (bc_force > 0) t.bc = std::min(t.bc, bc_force);  // (fused backward: the data path's chunks)
  t.nchunks = cdiv(B, t.bc);
  t.Kc = cdiv(2 * t.bc * t.T2, oaa::kTcK);
  // split-K for parallelism (≥ ~4 CTAs per SM); the splits are summed in fp64 by the
  // finalize kernel, and inside a split the GEMM drains its TMEM accumulator every
  // kTcDrain K chunks (oaa_tc.cuh).
  const int tiles = t.F * t.RTA * cdiv(2 * C, oaa::kTcM * t.NB);
  t.S = std::max(1, std::min(t.Kc, cdiv(4 * 148, tiles)));
  t.kps = cdiv(t.Kc, t.S);
  t.S = cdiv(t.Kc, t.kps);
  t.G = t.S;  // chunks accumulate into the same per-split slabs, in stream order
  t.SWg = cdiv(t.Td * t.BB, 4) * 4;
  t.SWx = cdiv(t.Td * t.BB + n - 1, 4) * 4;
  t.a_b = align_up(sizeof(float) * (size_t)t.F * t.Kc * t.RTA * 4096);
  t.b_b = align_up(sizeof(float) * (size_t)t.F * t.Kc * t.RTB * 4096);
  t.part_b = align_up(sizeof(float2) * (size_t)t.G * K * C * t.F);
  return t;
}

cudaError_t launch_filter_spectra(int n, const oaa::FiltSpecParams& p, bool xwin, int items, size_t smem,
                                  cudaStream_t s) {
  switch (n) {
    case 1: return launch_filter_spectra_n<1>(p, xwin, items, smem, s);
    case 2: return launch_filter_spectra_n<2>(p, xwin, items, smem, s);
    case 3: return launch_filter_spectra_n<3>(p, xwin, items, smem, s);
    case 4: return launch_filter_spectra_n<4>(p, xwin, items, smem, s);
    case 5: return launch_filter_spectra_n<5>(p, xwin, items, smem, s);
    case 6: return launch_filter_spectra_n<6>(p, xwin, items, smem, s);
    case 7: return launch_filter_spectra_n<7>(p, xwin, items, smem, s);
    case 8: return launch_filter_spectra_n<8>(p, xwin, items, smem, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_bin_gemm(const oaa::BinGemmParams& p, cudaStream_t s) {
  const bool conv = !(p.a_split && p.b_split);
  auto k = conv ? oaa::oaa_bin_gemm_kernel<true> : oaa::oaa_bin_gemm_kernel<false>;
  cudaError_t err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)oaa::kTcSmem);
  if (err != cudaSuccess) return err;
  // persistent: one CTA per SM (512 TMEM columns, 192 KB of stages), tiles strided over them
  const long long ntiles = (long long)cdiv(p.N, oaa::kTcM * p.NB) * cdiv(p.M, oaa::kTcM) * p.F * p.S;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)std::max<long long>(1, std::min<long long>(ntiles, sms));
  {
    KTimer kt(KID_BIN_GEMM, s);
    k<<<grid, conv ? oaa::tc_threads<true>() : oaa::tc_threads<false>(), oaa::kTcSmem, s>>>(p);
  }
  g_launches++;
  return cudaGetLastError();
}

// Tensor-core evaluation of fwd / bwd_data: per batch chunk, T1 (tile spectra) → bin
// GEMM (3×TF32 tcgen05) → walker in load mode (inverse DFT + overlap-add + crop).
struct TcData {
  oaa::TileSpecParams tp;
  oaa::BinGemmParams gp;
  oaa::WalkParams wp;
  size_t t1_smem, walk_smem;
  int n, T;
  long long F;
};
oaa_status_t tc_data_setup(TcData& d, bool is_fwd, const float* in, const float* w, float* out, int K, int C, int n,
                           const Geo& g, const EnginePlan& e, const TcPlan& tc, float* Ag, float* Xg, float* D,
                           cudaStream_t s, const void* prepared) {
  const int Cin = e.Cin, Cout = e.Cout, T = tc.T;  // (tc.T = e.T for blocks of the kernel's size)
  if (!prepared) {
    if (cudaMemsetAsync(Ag, 0, tc.ag_b, s) != cudaSuccess) return OAA_ERR_CUDA;
    const long long total = (long long)tc.F * Cin * Cout;
    const int thr = 256;
    const int blocks = (int)std::min<long long>((total + thr - 1) / thr, 8192);
    KTimer kt(KID_SPECTRUM, s);
    oaa::oaa_realified_spectrum_kernel<<<blocks, thr, 0, s>>>(w, Ag, K, C, n, tc.P, is_fwd ? 0 : 1, tc.Kc, tc.RTA);
    g_launches++;
    if (cudaGetLastError() != cudaSuccess) return OAA_ERR_CUDA;
  }
  d.n = n;
  d.T = T;
  d.F = tc.F;
  const int BB = tc.BB, H = tc.H;
  const int BW = BB == n ? e.BW : cdiv(T * BB, 4) * 4;  // staged row width of the tile producer
  oaa::TileSpecParams& tp = d.tp;
  tp = oaa::TileSpecParams{};
  tp.in = in;
  tp.Xg = Xg;
  tp.Cin = Cin;
  tp.R = e.R;
  tp.T = T;
  tp.Kc = tc.Kc;
  tp.RTB = tc.RTB;
  tp.BW = BW;
  tp.CSTR = BB * BW + 4;
  tp.BB = BB;
  tp.split = tc.b_split ? 1 : 0;
  tp.Ga = nullptr;
  d.t1_smem = sizeof(float) * 16 * (size_t)tp.CSTR;
  oaa::BinGemmParams& gp = d.gp;
  gp = oaa::BinGemmParams{};
  gp.A = Ag;
  gp.B = Xg;
  gp.D = D;
  gp.F = tc.F;
  gp.M = 2 * Cout;
  gp.Kc = tc.Kc;
  gp.RTA = tc.RTA;
  gp.RTB = tc.RTB;
  gp.S = 1;
  gp.kps = tc.Kc;
  gp.mode = 2;  // Ŷ straight into the walker's chunk layout
  gp.a_split = 1;
  gp.b_split = tc.b_split ? 1 : 0;
  gp.partial = nullptr;
  gp.Cf = Cout;
  gp.H = H;
  gp.P = tc.P;
  gp.TT = T;
  gp.TPW = 32 / H;
  gp.NT4 = cdiv(T, gp.TPW);
  gp.SBL = oaa::kYSBL;  // (the walker's load mode reads Ŷ with this block size fixed at compile time)
  gp.SB = 1 << gp.SBL;
  gp.NB = tc.NB;
  gp.Kuse = tc.Kc;
  // walker in LOAD mode: inverse DFT + overlap-add of Ŷ straight from the GEMM output
  const int TPW = 32 / H, CW = TPW * BB;
  oaa::WalkParams& wp = d.wp;
  wp = oaa::WalkParams{};
  wp.out = out;
  wp.Cin = 0;
  wp.Cout = Cout;
  wp.T = T;
  wp.Ro = e.Ro;
  wp.off = e.off;
  wp.NCH = cdiv(e.off + e.Ro, CW);
  wp.KG = std::min(tc.P <= 11 ? 4 : 8, Cout);  // warps per load-walker CTA (oaa_walk.cuh launch bounds)
  wp.ngrp = cdiv(Cout, wp.KG);
  wp.D = D;
  wp.BB = BB;
  const int QSZ = ((2 * TPW + 1) * H * tc.P + 1) & ~1;
  d.walk_smem = sizeof(float2) * (size_t)wp.KG * QSZ + sizeof(float) * (size_t)wp.KG * oaa::walk_trp(n) * wp.NCH * CW;
  return OAA_OK;
}
// one batch chunk [b0, b0 + bc): operand producer, bin GEMM, walker
oaa_status_t tc_data_chunk(TcData& d, int b0, int bc, cudaStream_t s) {
  const int n = d.n, T = d.T;
  const long long btc = (long long)bc * T * T;
  d.tp.b0 = b0;
  d.tp.bc = bc;
  if (launch_tile_spectra(n, d.tp, d.t1_smem, s) != cudaSuccess) return OAA_ERR_CUDA;
  oaa::BinGemmParams& gp = d.gp;
  gp.N = (int)btc;
  gp.ldd = (int)btc;
  gp.strideD = (long long)gp.M * btc;
  gp.plane = ((long long)bc * T * gp.NT4 * gp.TPW + gp.SB - 1) / gp.SB * 2 * d.F * gp.SB;
  set_gemm_dmap(gp, ((long long)bc * T * gp.NT4 * gp.TPW + gp.SB - 1) / gp.SB);
  if (launch_bin_gemm(gp, s) != cudaSuccess) return OAA_ERR_CUDA;
  d.wp.B = bc;
  d.wp.b0 = b0;
  d.wp.BTc = (int)btc;
  d.wp.SBL = gp.SBL;
  if (launch_walk_load(n, d.wp, d.walk_smem, bc, s) != cudaSuccess) return OAA_ERR_CUDA;
  return OAA_OK;
}

oaa_status_t run_engine_tc(bool is_fwd, const float* in, const float* w, float* out, int B, int C, int K, int n,
                           const Geo& g, const EnginePlan& e, const TcPlan& tc, const EngineWs& L, char* base,
                           cudaStream_t s, const void* prepared) {
  float* Ag = prepared ? static_cast<float*>(const_cast<void*>(prepared)) : reinterpret_cast<float*>(base + L.spec_off);
  float* Xg = reinterpret_cast<float*>(base + L.xg_off);
  float* D = reinterpret_cast<float*>(base + L.d_off);
  TcData d;
  oaa_status_t st = tc_data_setup(d, is_fwd, in, w, out, K, C, n, g, e, tc, Ag, Xg, D, s, prepared);
  if (st != OAA_OK) return st;
  ProfScope prof(is_fwd ? OAA_OP_FWD : OAA_OP_BWD_DATA, s);
  prof.start();
  for (int b0 = 0; b0 < B; b0 += tc.bc)
    if ((st = tc_data_chunk(d, b0, std::min(tc.bc, B - b0), s)) != OAA_OK) return st;
  prof.stop();
  return OAA_OK;
}

// prepared != NULL: the weight spectra were computed by oaa_weight_spectra (cached across
// calls, NEXT-4 of SURVEY.md §8(f)); w is then unused and may be NULL
oaa_status_t run_engine(bool is_fwd, const float* in, const float* w, float* out, int B, int C,
                        int K, int N, int n, oaa_crop_t crop, void* ws, size_t ws_bytes,
                        void* stream, const void* prepared = nullptr) {
  Geo g;
  oaa_status_t st = validate(B, C, K, N, n, crop, &g);
  if (st != OAA_OK) return st;
  if ((!w && !prepared) || (B > 0 && (!in || !out))) return OAA_ERR_INVALID_VALUE;
  if (prepared && (reinterpret_cast<uintptr_t>(prepared) % kAlign) != 0) return OAA_ERR_INVALID_VALUE;
  const int R = is_fwd ? N : g.M, Ro = is_fwd ? g.M : N;
  const int Cin = is_fwd ? C : K, Cout = is_fwd ? K : C;
  const int off = is_fwd ? g.o : (n - 1 - g.o);
  const size_t in_bytes = sizeof(float) * (size_t)B * Cin * R * R;
  const size_t out_bytes = sizeof(float) * (size_t)B * Cout * Ro * Ro;
  const size_t w_bytes = sizeof(float) * (size_t)K * C * n * n;
  if (B > 0 && (overlaps(in, in_bytes, out, out_bytes) || (w && overlaps(w, w_bytes, out, out_bytes))))
    return OAA_ERR_INVALID_VALUE;
  const TcPlan tc = plan_tc(B, Cin, Cout, R, n);
  EnginePlan e;
  if (!plan_engine(R, Ro, off, n, Cin, Cout, &e, tc.use)) return OAA_ERR_UNSUPPORTED;
  if (B == 0) return OAA_OK;
  const WalkHostGeo wk = plan_walk(is_fwd, B, Cin, Cout, R, Ro, off, n, tc);
  const BwddPlan bd = plan_bwdd(is_fwd, B, Cout, R, n, tc);
  EngineWs L = engine_ws(B, C, K, e.T, g, tc, &wk, &bd);
  if (!ws || ws_bytes < L.total || (reinterpret_cast<uintptr_t>(ws) % kAlign) != 0)
    return OAA_ERR_WORKSPACE;
  if (overlaps(ws, L.total, out, out_bytes) || overlaps(ws, L.total, in, in_bytes) ||
      (w && overlaps(ws, L.total, w, w_bytes)))
    return OAA_ERR_INVALID_VALUE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  char* base = static_cast<char*>(ws);
  float4* spec = prepared ? static_cast<float4*>(const_cast<void*>(prepared))
                          : reinterpret_cast<float4*>(base + L.spec_off);
  int* flags = reinterpret_cast<int*>(base + L.flags_off);
  int* counter = reinterpret_cast<int*>(base + L.counter_off);

  if (tc.use) return run_engine_tc(is_fwd, in, w, out, B, C, K, n, g, e, tc, L, base, s, prepared);
  if (bd.use) {
    ProfScope prof(OAA_OP_BWD_DATA, s);
    prof.start();
    if (cudaMemsetAsync(out, 0, out_bytes, s) != cudaSuccess) return OAA_ERR_CUDA;
    if (!prepared) {
      KTimer kt(KID_SPECTRUM, s);
      oaa::oaa_spectrum_kernel<<<K * C, 128, 0, s>>>(w, spec, K, C, n, bd.P, 1, 1);
      g_launches++;
      if (cudaGetLastError() != cudaSuccess) return OAA_ERR_CUDA;
    }
    oaa::BwdDParams dp;
    dp.dy = in;
    dp.spec = spec;
    dp.dx = out;
    dp.B = B;
    dp.K = K;
    dp.C = C;
    dp.M = R;
    dp.N = Ro;
    dp.Td = bd.Td;
    dp.off = off;
    dp.NCW = bd.NCW;
    dp.RPC = bd.RPC;
    dp.WSL = bd.WSL;
    dp.BB = bd.BB;
    cudaError_t err = launch_bwdd(n, dp, C, bd.smem, s);
    prof.stop();
    return err == cudaSuccess ? OAA_OK : OAA_ERR_CUDA;
  }
  if (wk.use) {
    if (!prepared) {
      KTimer kt(KID_SPECTRUM, s);
      oaa::oaa_spectrum_kernel<<<K * C, 128, 0, s>>>(w, spec, K, C, n, wk.P, 0, 1);
      g_launches++;
      if (cudaGetLastError() != cudaSuccess) return OAA_ERR_CUDA;
    }
    oaa::XSpecParams xp;
    xp.in = in;
    xp.S = reinterpret_cast<float4*>(base + L.xg_off);
    xp.Cin = Cin;
    xp.R = R;
    xp.T = wk.T;
    xp.NCH = wk.NCH;
    xp.SW = wk.NCH * wk.CW;
    xp.org = 0;
    set_xspec_tma(xp, B, wk.BB);
    oaa::WalkParams wp;
    wp.S = xp.S;
    wp.spec = spec;
    wp.out = out;
    wp.B = B;
    wp.Cin = Cin;
    wp.Cout = Cout;
    wp.T = wk.T;
    wp.Ro = Ro;
    wp.off = off;
    wp.NCH = wk.NCH;
    wp.KG = wk.KG;
    wp.ngrp = wk.ngrp;
    WalkPlan wpl;
    wpl.KG = wk.KG;
    wpl.ngrp = wk.ngrp;
    wpl.NCH = wk.NCH;
    wpl.SW = xp.SW;
    wpl.BB = wk.BB;
    wpl.xspec_smem = oaa::xspec_smem_bytes(Cin, wk.BB, xp.SW, wk.CH4);
    const int QSZ = ((2 * wk.TPW + 1) * wk.H * wk.P + 1) & ~1;
    wpl.walk_smem = sizeof(float4) * (size_t)oaa::kWalkRing * Cin * wk.CH4 + sizeof(float2) * (size_t)wk.KG * QSZ +
                    sizeof(float) * (size_t)wk.KG * oaa::walk_trp(n) * wk.NCH * wk.CW;
    if (wpl.walk_smem > 220 * 1024 || wpl.xspec_smem > 220 * 1024) return OAA_ERR_UNSUPPORTED;
    ProfScope prof(OAA_OP_FWD, s);
    prof.start();
    cudaError_t err = launch_walk(n, xp, wp, wpl, Cin, s);
    prof.stop();
    return err == cudaSuccess ? OAA_OK : OAA_ERR_CUDA;
  }
  // kernel spectra: loop-major layout [Cloop][Cinner][P][H]
  const int loop_is_k = (is_fwd == e.S1) ? 1 : 0;  // fwd S1 / bwd_data S2 loop over k
  if (!prepared) {
    KTimer kt(KID_SPECTRUM, s);
    oaa::oaa_spectrum_kernel<<<K * C, 128, 0, s>>>(w, spec, K, C, n, 2 * n - 1, is_fwd ? 0 : 1, loop_is_k);
    g_launches++;
    if (cudaGetLastError() != cudaSuccess) return OAA_ERR_CUDA;
  }
  if (cudaMemsetAsync(base + L.flags_off, 0, L.total - L.flags_off, s) != cudaSuccess)
    return OAA_ERR_CUDA;
  oaa::EngineParams p;
  p.in = in;
  p.spec = spec;
  p.out = out;
  p.flags = flags;
  p.counter = counter;
  p.B = B;
  p.Cin = Cin;
  p.Cout = Cout;
  p.R = R;
  p.T = e.T;
  p.Ro = Ro;
  p.off = off;
  p.TS = e.TS;
  p.BW = e.BW;
  p.num_items = B * e.T;
  p.ncomp = e.ncomp;
  p.CIG = e.CIG;
  ProfScope prof(is_fwd ? OAA_OP_FWD : OAA_OP_BWD_DATA, s);
  prof.start();
  cudaError_t err = launch_engine(n, p, e, s);
  prof.stop();
  return err == cudaSuccess ? OAA_OK : OAA_ERR_CUDA;
}

// tensor-core weight gradient: per batch chunk the Ĝ / Ξ̂ operand spectra, then the split-K
// bin GEMM accumulating per-split partial dŴ; after the last chunk the fp64 finalize
struct TcFilt {
  oaa::FiltSpecParams gs, xs;
  oaa::BinGemmParams gp;
  size_t smem_g, smem_x;
  TcFiltPlan t;
  float *Ga, *Xb, *part;
  int n;
};
void tc_filt_setup(TcFilt& f, const float* x, const float* dy, int C, int K, int N, int n, const Geo& g,
                   const TcFiltPlan& t, char* base) {
  f.t = t;
  f.n = n;
  f.Ga = reinterpret_cast<float*>(base);
  f.Xb = reinterpret_cast<float*>(base + t.a_b);
  f.part = reinterpret_cast<float*>(base + t.a_b + t.b_b);
  f.gs = oaa::FiltSpecParams{};
  f.gs.src = dy; f.gs.Op = f.Ga; f.gs.nch = K; f.gs.R = g.M; f.gs.Td = t.Td; f.gs.org = 0; f.gs.Kc = t.Kc;
  f.gs.RT = t.RTA; f.gs.SW = t.SWg;
  f.xs = oaa::FiltSpecParams{};
  f.xs.src = x; f.xs.Op = f.Xb; f.xs.nch = C; f.xs.R = N; f.xs.Td = t.Td; f.xs.org = g.o - (n - 1); f.xs.Kc = t.Kc;
  f.xs.RT = t.RTB; f.xs.SW = t.SWx;
  f.gs.BB = t.BB;
  f.xs.BB = t.BB;
  f.smem_g = 2 * sizeof(float) * oaa::kFsCG * t.BB * (size_t)t.SWg;  // double-buffered bands
  f.smem_x = 2 * sizeof(float) * oaa::kFsCG * t.P * (size_t)t.SWx;
  oaa::BinGemmParams& gp = f.gp;
  gp = oaa::BinGemmParams{};
  gp.A = f.Ga; gp.B = f.Xb; gp.D = nullptr; gp.F = t.F; gp.M = K; gp.N = 2 * C; gp.Kc = t.Kc; gp.RTA = t.RTA;
  gp.RTB = t.RTB; gp.ldd = 0; gp.strideD = 0; gp.S = t.S; gp.kps = t.kps; gp.mode = 1; gp.a_split = 0; gp.Cf = C;
  gp.H = t.H; gp.P = t.P; gp.partial = f.part; gp.NB = t.NB;
}
// chunk ci = images [b0, b0 + bc); g_done: Ĝ already written by the fused dy producer
oaa_status_t tc_filt_chunk(TcFilt& f, int ci, int b0, int bc, bool g_done, cudaStream_t s) {
  const TcFiltPlan& t = f.t;
  const int n = f.n;
  f.gs.b0 = b0;
  f.xs.b0 = b0;
  if (!g_done && launch_filter_spectra(n, f.gs, false, bc * t.Td, f.smem_g, s) != cudaSuccess) return OAA_ERR_CUDA;
  if (launch_filter_spectra(n, f.xs, true, bc * t.Td, f.smem_x, s) != cudaSuccess) return OAA_ERR_CUDA;
  // a short last chunk: the GEMM reduces only the K chunks holding data, and only the
  // ragged end of the last one is zeroed
  const int j0 = 2 * bc * t.T2;
  f.gp.Kuse = cdiv(j0, oaa::kTcK);
  if (j0 < 32 * f.gp.Kuse) {
    KTimer kt(KID_AUX, s);
    oaa::oaa_tc_zero_tail_kernel<<<512, 256, 0, s>>>(f.Ga, t.F, t.Kc, t.RTA, j0, 32 * f.gp.Kuse);
    oaa::oaa_tc_zero_tail_kernel<<<512, 256, 0, s>>>(f.Xb, t.F, t.Kc, t.RTB, j0, 32 * f.gp.Kuse);
    g_launches += 2;
    if (cudaGetLastError() != cudaSuccess) return OAA_ERR_CUDA;
  }
  f.gp.g0 = 0;
  f.gp.accumulate = ci > 0;
  return launch_bin_gemm(f.gp, s) == cudaSuccess ? OAA_OK : OAA_ERR_CUDA;
}
// fp64 finalize of the weight gradient: many partial spectra (the SIMT kernels' G ≈ 148
// slices) → one 512-thread CTA per (k, c) with the sum spread over 4 × bins threads; few
// (the tensor-core splits) → one warp per (k, c), 8 per CTA.
// P: transform size of the partial spectra (2n − 1, or b + n − 1 for blocks b ≠ n)
void launch_finalize(const float2* partial, float* dw, int G, int K, int C, int n, cudaStream_t s, int P = 0) {
  KTimer kt(KID_FINALIZE, s);
  if (P == 0) P = 2 * n - 1;
  if (G >= 32)
    oaa::oaa_filter_finalize_kernel<<<K * C, 512, sizeof(double2) * P * ((P + 1) / 2), s>>>(partial, dw, G, K, C, n, P);
  else
    oaa::oaa_filter_finalize_small_kernel<<<(K * C + 7) / 8, 256, 0, s>>>(partial, dw, G, K, C, n, P);
}
oaa_status_t tc_filt_finalize(TcFilt& f, float* dw, int K, int C, cudaStream_t s) {
  launch_finalize(reinterpret_cast<const float2*>(f.part), dw, f.t.G, K, C, f.n, s, f.t.P);
  g_launches++;
  return cudaGetLastError() == cudaSuccess ? OAA_OK : OAA_ERR_CUDA;
}

oaa_status_t run_filter_tc(const float* x, const float* dy, float* dw, int B, int C, int K, int N, int n,
                           const Geo& g, const TcFiltPlan& t, void* ws, size_t ws_bytes, cudaStream_t s,
                           size_t x_bytes, size_t dy_bytes, size_t dw_bytes) {
  const size_t need = t.a_b + t.b_b + t.part_b;
  if (!ws || ws_bytes < need || (reinterpret_cast<uintptr_t>(ws) % kAlign) != 0) return OAA_ERR_WORKSPACE;
  if (overlaps(ws, need, dw, dw_bytes) || overlaps(ws, need, x, x_bytes) || overlaps(ws, need, dy, dy_bytes))
    return OAA_ERR_INVALID_VALUE;
  TcFilt f;
  tc_filt_setup(f, x, dy, C, K, N, n, g, t, static_cast<char*>(ws));
  ProfScope prof(OAA_OP_BWD_FILTER, s);
  prof.start();
  for (int ci = 0; ci < t.nchunks; ++ci) {
    const int b0 = ci * t.bc;
    oaa_status_t st = tc_filt_chunk(f, ci, b0, std::min(t.bc, B - b0), false, s);
    if (st != OAA_OK) return st;
  }
  prof.stop();
  return tc_filt_finalize(f, dw, K, C, s);
}

cudaError_t launch_bwd_fused(int n, const oaa::XSpecParams& xp, const oaa::BwdDParams& pd, const oaa::BwdFParams& pf,
                             size_t xsmem, size_t smem, int nf, cudaStream_t s) {
  switch (n) {
    case 1: return launch_bwd_fused_n<1>(xp, pd, pf, xsmem, smem, nf, s);
    case 2: return launch_bwd_fused_n<2>(xp, pd, pf, xsmem, smem, nf, s);
    case 3: return launch_bwd_fused_n<3>(xp, pd, pf, xsmem, smem, nf, s);
    case 4: return launch_bwd_fused_n<4>(xp, pd, pf, xsmem, smem, nf, s);
    case 5: return launch_bwd_fused_n<5>(xp, pd, pf, xsmem, smem, nf, s);
    case 6: return launch_bwd_fused_n<6>(xp, pd, pf, xsmem, smem, nf, s);
    case 7: return launch_bwd_fused_n<7>(xp, pd, pf, xsmem, smem, nf, s);
    case 8: return launch_bwd_fused_n<8>(xp, pd, pf, xsmem, smem, nf, s);
  }
  return cudaErrorInvalidValue;
}

// fused backward (NEXT-1): both backward convolutions of PAPER.md:89 in one call.  On the
// tensor-core path the dy-block spectra Ĝ are computed ONCE per batch chunk and written
// both as the data-gradient GEMM's B operand and as the weight-gradient GEMM's A operand
// (dy read once, one set of dy FFTs); elsewhere the two ops run back to back.
struct BwdFusedPlan {
  bool tc;
  bool simt;  // one launch of both SIMT bodies (oaa_bwd_fused_kernel)
  TcPlan td;
  TcFiltPlan tf;
  EnginePlan e;
  BwddPlan bd;
  BwdfPlan bf;  // with G = one weight-gradient CTA per SM (nf = G·nkg CTAs)
  size_t data_b, filt_b, total, smem;
};
bool plan_bwd_fused(int B, int C, int K, int N, int n, oaa_crop_t crop, const Geo& g, BwdFusedPlan* p) {
  *p = BwdFusedPlan{};
  p->td = plan_tc(B, K, C, g.M, n);
  TcFiltPlan tf0 = plan_tc_filter(B, C, K, N, g.M, n);
  p->tc = p->td.use && tf0.use && B > 0;
  if (p->tc) {
    if (!plan_engine(g.M, N, n - 1 - g.o, n, K, C, &p->e, true)) return false;
    p->tf = plan_tc_filter(B, C, K, N, g.M, n, p->td.bc, p->td.BB);
    p->data_b = align_up(engine_ws(B, C, K, p->e.T, g, p->td).total);
    p->filt_b = align_up(p->tf.a_b + p->tf.b_b + p->tf.part_b);
  } else {
    p->data_b = align_up(oaa_conv_workspace_bytes(OAA_OP_BWD_DATA, B, C, K, N, n, crop));
    p->filt_b = align_up(oaa_conv_workspace_bytes(OAA_OP_BWD_FILTER, B, C, K, N, n, crop));
    // SIMT family: both bodies fit 128 registers, ≤ 110 KB of shared memory and 256 TMEM
    // columns, and the weight-gradient CTA has the full 8 warps
    const TcPlan none{};
    p->bd = plan_bwdd(false, B, C, g.M, n, none);
    p->bf = plan_bwdf(B, C, K, g.M, n);
    const size_t bsm = oaa::bwdd_smem_bytes(n, p->bd.BB, C, p->bd.NCW, p->bd.RPC, p->bd.WSL);
    p->simt = B > 0 && p->bd.use && p->bf.use && p->bf.nwb == oaa::kBwdfWarps && bsm <= 110 * 1024 &&
              p->bf.smem <= 110 * 1024;
    if (p->simt) {
#ifndef OAA_EXP_FUSED_SLOTS  // experiment builds only: -DOAA_EXP_FUSED_SLOTS=<weight-gradient CTAs>
#define OAA_EXP_FUSED_SLOTS 296  // measured: 74 → 3.45, 148 → 2.75, 222 → 2.73, 296 → 2.72 ms (headline)
#endif
      p->bf.G = std::max(1, std::min(B * p->bf.Td, OAA_EXP_FUSED_SLOTS / p->bf.nkg));
      p->bf.part_b = align_up(sizeof(float2) * (size_t)p->bf.G * K * C * (2 * n - 1) * n);
      p->smem = std::max(bsm, p->bf.smem);
      p->data_b = align_up(sizeof(float4) * (size_t)K * C * n * n);
      p->filt_b = p->bf.xs_b + p->bf.part_b;
    }
  }
  p->total = p->data_b + p->filt_b;
  return true;
}

// Overlap-and-save forward on the tensor-core path (C, K ≥ 16; NEXT-2): per
// batch chunk the spectra of the (2n−1)² x-windows of the OUTPUT tiles (tile spectra, window
// mode), the bin GEMM, and the walker in load + overlap-and-save mode (the blocks' last n rows
// and columns, no overlap-add).  Workspace: the tensor-core engine's layout over ⌈M/n⌉² tiles.
struct OasTc {
  bool use;
  TcPlan tc;
  EnginePlan e;
  EngineWs L;
};
OasTc plan_oas_tc(int B, int C, int K, int N, int n, const Geo& g) {
  OasTc o{};
  o.tc = plan_tc(B, C, K, g.M, n, false);  // tiles: ⌈M/n⌉² output tiles
  o.use = o.tc.use && B > 0;
  if (!o.use) return o;
  o.e = EnginePlan{};
  o.e.R = N;  // the windows read x
  o.e.Ro = g.M;
  o.e.off = 0;
  o.e.T = cdiv(g.M, n);
  o.e.Cin = C;
  o.e.Cout = K;
  o.e.BW = cdiv(o.e.T * n + n - 1, 4) * 4;
  o.L = engine_ws(B, C, K, o.e.T, g, o.tc);
  return o;
}
oaa_status_t run_oas_tc(const float* x, const float* w, float* y, int B, int C, int K, int n, const Geo& g,
                        const OasTc& o, char* base, cudaStream_t s) {
  float* Ag = reinterpret_cast<float*>(base + o.L.spec_off);
  float* Xg = reinterpret_cast<float*>(base + o.L.xg_off);
  float* D = reinterpret_cast<float*>(base + o.L.d_off);
  TcData d;
  oaa_status_t st = tc_data_setup(d, true, x, w, y, K, C, n, g, o.e, o.tc, Ag, Xg, D, s, nullptr);
  if (st != OAA_OK) return st;
  const int P = 2 * n - 1;
  d.tp.win = 1;
  d.tp.org = g.o - (n - 1);
  d.tp.CSTR = P * d.tp.BW + 4;
  d.t1_smem = sizeof(float) * 4 * (size_t)d.tp.CSTR;
  d.wp.oas = 1;
  ProfScope prof(OAA_OP_FWD, s);
  prof.start();
  for (int b0 = 0; b0 < B; b0 += o.tc.bc)
    if ((st = tc_data_chunk(d, b0, std::min(o.tc.bc, B - b0), s)) != OAA_OK) return st;
  prof.stop();
  return OAA_OK;
}

}  // namespace

extern "C" {

int oaa_conv_out_size(int N, int n, oaa_crop_t crop) {
  if (N < 1 || n < 1) return -1;
  switch (crop) {
    case OAA_CROP_FULL: return N + n - 1;
    case OAA_CROP_VALID: return n <= N ? N - n + 1 : -1;
    case OAA_CROP_SAME: return N;
  }
  return -1;
}

size_t oaa_conv_workspace_bytes(oaa_op_t op, int B, int C, int K, int N, int n, oaa_crop_t crop) {
  Geo g;
  if (validate(B, C, K, N, n, crop, &g) != OAA_OK) return 0;
  if (B == 0) return 0;
  if (op == OAA_OP_FWD || op == OAA_OP_BWD_DATA) {
    const bool fwd = op == OAA_OP_FWD;
    const int R = fwd ? N : g.M;
    const TcPlan tc = plan_tc(B, fwd ? C : K, fwd ? K : C, R, n);
    const int Ro = fwd ? g.M : N, off = fwd ? g.o : (n - 1 - g.o);
    const WalkHostGeo wk = plan_walk(fwd, B, fwd ? C : K, fwd ? K : C, R, Ro, off, n, tc);
    const BwddPlan bd = plan_bwdd(fwd, B, fwd ? K : C, R, n, tc);
    return engine_ws(B, C, K, cdiv(R, n), g, tc, &wk, &bd).total;
  }
  if (op == OAA_OP_BWD) {
    BwdFusedPlan fp;
    if (!plan_bwd_fused(B, C, K, N, n, crop, g, &fp)) return 0;
    return fp.total;
  }
  if (op == OAA_OP_FWD_OAS) {
    const OasPlan o = plan_oas(B, C, K, N, n, g);
    if (o.use) return o.spec_b + o.xs_b;
    const OasTc ot = plan_oas_tc(B, C, K, N, n, g);
    return ot.use ? ot.L.total : 0;
  }
  if (op == OAA_OP_BWD_FILTER) {
    const TcFiltPlan t = plan_tc_filter(B, C, K, N, g.M, n);
    if (t.use) return t.a_b + t.b_b + t.part_b;
    const BwdfPlan bf = plan_bwdf(B, C, K, g.M, n);
    if (bf.use) return bf.xs_b + bf.part_b;
    FilterPlan f;
    if (!plan_filter(B, C, K, g.M, n, &f)) return 0;
    return align_up(sizeof(float2) * (size_t)f.G * K * C * g.P * g.H);
  }
  return 0;
}

// Prepared weight spectra ("a caller-visible 'prepared
// kernel' cache ... for layer-level reuse across many inputs"): the spectra a fwd /
// bwd_data call with these arguments computes first, written once into a caller buffer.
struct SpecPlan {
  bool ok;
  size_t bytes;
};
SpecPlan spec_plan(bool is_fwd, int C, int K, int N, int n, const Geo& g) {
  SpecPlan sp{};
  const int R = is_fwd ? N : g.M, Ro = is_fwd ? g.M : N;
  const int Cin = is_fwd ? C : K, Cout = is_fwd ? K : C;
  const int off = is_fwd ? g.o : (n - 1 - g.o);
  const TcPlan tc = plan_tc(1, Cin, Cout, R, n);
  EnginePlan e;
  if (!plan_engine(R, Ro, off, n, Cin, Cout, &e, tc.use)) return sp;
  const WalkHostGeo wk = plan_walk(is_fwd, 1, Cin, Cout, R, Ro, off, n, tc);
  const BwddPlan bd = plan_bwdd(is_fwd, 1, Cout, R, n, tc);
  sp.ok = true;
  // the TC path's real-ified, pre-split UMMA-blocked weights, else the float4 bin-pair
  // spectra [.][.][n][n] of the engine kernels ([.][.][H][H] for the walker and bwd_data,
  // whose blocks may be larger than n)
  sp.bytes = tc.use   ? align_up(tc.ag_b)
             : wk.use ? wk.spec_b
             : bd.use ? align_up(sizeof(float4) * (size_t)K * C * bd.H * bd.H)
                      : align_up(sizeof(float4) * (size_t)K * C * n * n);
  return sp;
}

oaa_status_t oaa_conv_fwd(const float* x, const float* w, float* y, int B, int C, int K, int N,
                          int n, oaa_crop_t crop, void* ws, size_t ws_bytes, void* stream) {
  return run_engine(true, x, w, y, B, C, K, N, n, crop, ws, ws_bytes, stream);
}

oaa_status_t oaa_conv_bwd(const float* x, const float* dy, const float* w, float* dx, float* dw, int B, int C,
                          int K, int N, int n, oaa_crop_t crop, void* ws, size_t ws_bytes, void* stream) {
  Geo g;
  oaa_status_t st = validate(B, C, K, N, n, crop, &g);
  if (st != OAA_OK) return st;
  if (!w || !dw || (B > 0 && (!x || !dy || !dx))) return OAA_ERR_INVALID_VALUE;
  const size_t x_bytes = sizeof(float) * (size_t)B * C * N * N;
  const size_t dy_bytes = sizeof(float) * (size_t)B * K * g.M * g.M;
  const size_t w_bytes = sizeof(float) * (size_t)K * C * n * n;
  if (overlaps(dx, x_bytes, dw, w_bytes) || overlaps(dx, x_bytes, dy, dy_bytes) || overlaps(dx, x_bytes, x, x_bytes) ||
      overlaps(dx, x_bytes, w, w_bytes) || overlaps(dw, w_bytes, x, x_bytes) || overlaps(dw, w_bytes, dy, dy_bytes) ||
      overlaps(dw, w_bytes, w, w_bytes))
    return OAA_ERR_INVALID_VALUE;
  BwdFusedPlan fp;
  if (!plan_bwd_fused(B, C, K, N, n, crop, g, &fp)) return OAA_ERR_UNSUPPORTED;
  char* base = static_cast<char*>(ws);
  if (fp.simt) {  // one launch of both SIMT bodies
    if (!ws || ws_bytes < fp.total || (reinterpret_cast<uintptr_t>(ws) % kAlign) != 0) return OAA_ERR_WORKSPACE;
    if (overlaps(ws, fp.total, dx, x_bytes) || overlaps(ws, fp.total, dw, w_bytes) ||
        overlaps(ws, fp.total, x, x_bytes) || overlaps(ws, fp.total, dy, dy_bytes) || overlaps(ws, fp.total, w, w_bytes))
      return OAA_ERR_INVALID_VALUE;
    if (std::max(cdiv(N, n) * n, g.M) > oaa::kMaxThreads) return OAA_ERR_UNSUPPORTED;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    float4* spec = reinterpret_cast<float4*>(base);
    const BwdfPlan& bf = fp.bf;
    if (cudaMemsetAsync(dx, 0, x_bytes, s) != cudaSuccess) return OAA_ERR_CUDA;
    {
      KTimer kt(KID_SPECTRUM, s);
      oaa::oaa_spectrum_kernel<<<K * C, 128, 0, s>>>(w, spec, K, C, n, fp.bd.P, 1, 1);
      g_launches++;
      if (cudaGetLastError() != cudaSuccess) return OAA_ERR_CUDA;
    }
    oaa::BwdDParams dp;
    dp.dy = dy; dp.spec = spec; dp.dx = dx; dp.B = B; dp.K = K; dp.C = C; dp.M = g.M; dp.N = N;
    dp.Td = fp.bd.Td; dp.off = n - 1 - g.o; dp.NCW = fp.bd.NCW;
    dp.RPC = fp.bd.RPC; dp.WSL = fp.bd.WSL; dp.BB = fp.bd.BB;
    oaa::XSpecParams xp;
    xp.in = x; xp.S = reinterpret_cast<float4*>(base + fp.data_b); xp.Cin = C; xp.R = N; xp.T = bf.Td;
    xp.NCH = bf.NCH; xp.SW = bf.SW; xp.org = g.o - (n - 1);
    set_xspec_tma(xp, B, 2 * n - 1);
    oaa::BwdFParams pf;
    pf.dy = dy; pf.XS = xp.S; pf.partial = reinterpret_cast<float2*>(base + fp.data_b + bf.xs_b); pf.B = B; pf.K = K;
    pf.C = C; pf.M = g.M; pf.Td = bf.Td; pf.NCH = bf.NCH; pf.G = bf.G; pf.KG = bf.KG;
    if (launch_bwd_fused(n, xp, dp, pf, bf.xspec_smem, fp.smem, bf.G * bf.nkg, s) != cudaSuccess) return OAA_ERR_CUDA;
    launch_finalize(pf.partial, dw, bf.G, K, C, n, s);
    g_launches++;
    return cudaGetLastError() == cudaSuccess ? OAA_OK : OAA_ERR_CUDA;
  }
  if (!fp.tc) {  // the two ops back to back, each with its own part of the workspace
    if (B > 0 && (!ws || ws_bytes < fp.total || (reinterpret_cast<uintptr_t>(ws) % kAlign) != 0))
      return OAA_ERR_WORKSPACE;
    st = oaa_conv_bwd_filter(x, dy, dw, B, C, K, N, n, crop, B > 0 ? base + fp.data_b : ws, fp.filt_b, stream);
    if (st != OAA_OK) return st;
    return oaa_conv_bwd_data(dy, w, dx, B, C, K, N, n, crop, ws, fp.data_b, stream);
  }
  if (std::max(cdiv(N, n) * n, g.M) > oaa::kMaxThreads) return OAA_ERR_UNSUPPORTED;
  if (!ws || ws_bytes < fp.total || (reinterpret_cast<uintptr_t>(ws) % kAlign) != 0) return OAA_ERR_WORKSPACE;
  if (overlaps(ws, fp.total, dx, x_bytes) || overlaps(ws, fp.total, dw, w_bytes) || overlaps(ws, fp.total, x, x_bytes) ||
      overlaps(ws, fp.total, dy, dy_bytes) || overlaps(ws, fp.total, w, w_bytes))
    return OAA_ERR_INVALID_VALUE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const EngineWs L = engine_ws(B, C, K, fp.e.T, g, fp.td);
  TcData d;
  st = tc_data_setup(d, false, dy, w, dx, K, C, n, g, fp.e, fp.td, reinterpret_cast<float*>(base + L.spec_off),
                     reinterpret_cast<float*>(base + L.xg_off), reinterpret_cast<float*>(base + L.d_off), s, nullptr);
  if (st != OAA_OK) return st;
  TcFilt f;
  tc_filt_setup(f, x, dy, C, K, N, n, g, fp.tf, base + fp.data_b);
  d.tp.Ga = f.Ga;  // the dy producer also writes the weight-gradient operand
  d.tp.KcG = fp.tf.Kc;
  d.tp.RTG = fp.tf.RTA;
  const int bc = fp.tf.bc;  // ≤ the data path's chunk (plan_bwd_fused)
  for (int ci = 0; ci * bc < B; ++ci) {
    const int b0 = ci * bc, bcc = std::min(bc, B - b0);
    if ((st = tc_data_chunk(d, b0, bcc, s)) != OAA_OK) return st;
    if ((st = tc_filt_chunk(f, ci, b0, bcc, true, s)) != OAA_OK) return st;
  }
  return tc_filt_finalize(f, dw, K, C, s);
}

oaa_status_t oaa_conv_fwd_oas(const float* x, const float* w, float* y, int B, int C, int K, int N, int n,
                              oaa_crop_t crop, void* ws, size_t ws_bytes, void* stream) {
  Geo g;
  oaa_status_t st = validate(B, C, K, N, n, crop, &g);
  if (st != OAA_OK) return st;
  if (!w || (B > 0 && (!x || !y))) return OAA_ERR_INVALID_VALUE;
  const size_t x_bytes = sizeof(float) * (size_t)B * C * N * N;
  const size_t y_bytes = sizeof(float) * (size_t)B * K * g.M * g.M;
  const size_t w_bytes = sizeof(float) * (size_t)K * C * n * n;
  if (B > 0 && (overlaps(x, x_bytes, y, y_bytes) || overlaps(w, w_bytes, y, y_bytes))) return OAA_ERR_INVALID_VALUE;
  if (std::max(cdiv(N, n) * n, g.M) > oaa::kMaxThreads) return OAA_ERR_UNSUPPORTED;
  const OasPlan o = plan_oas(B, C, K, N, n, g);
  if (!o.use) {
    const OasTc ot = plan_oas_tc(B, C, K, N, n, g);
    if (B == 0 && plan_tc(1, C, K, g.M, n).use) return OAA_OK;
    if (!ot.use) return OAA_ERR_UNSUPPORTED;
    if (!ws || ws_bytes < ot.L.total || (reinterpret_cast<uintptr_t>(ws) % kAlign) != 0) return OAA_ERR_WORKSPACE;
    if (overlaps(ws, ot.L.total, y, y_bytes) || overlaps(ws, ot.L.total, x, x_bytes) ||
        overlaps(ws, ot.L.total, w, w_bytes))
      return OAA_ERR_INVALID_VALUE;
    return run_oas_tc(x, w, y, B, C, K, n, g, ot, static_cast<char*>(ws), static_cast<cudaStream_t>(stream));
  }
  if (B == 0) return OAA_OK;
  const size_t need = o.spec_b + o.xs_b;
  if (!ws || ws_bytes < need || (reinterpret_cast<uintptr_t>(ws) % kAlign) != 0) return OAA_ERR_WORKSPACE;
  if (overlaps(ws, need, y, y_bytes) || overlaps(ws, need, x, x_bytes) || overlaps(ws, need, w, w_bytes))
    return OAA_ERR_INVALID_VALUE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  char* base = static_cast<char*>(ws);
  float4* spec = reinterpret_cast<float4*>(base);
  ProfScope prof(OAA_OP_FWD, s);
  prof.start();
  {
    KTimer kt(KID_SPECTRUM, s);
    oaa::oaa_spectrum_kernel<<<K * C, 128, 0, s>>>(w, spec, K, C, n, 2 * n - 1, 0, 1);
    g_launches++;
    if (cudaGetLastError() != cudaSuccess) return OAA_ERR_CUDA;
  }
  oaa::XSpecParams xp;
  xp.in = x;
  xp.S = reinterpret_cast<float4*>(base + o.spec_b);
  xp.Cin = C;
  xp.R = N;
  xp.T = o.Td;
  xp.NCH = o.NCH;
  xp.SW = o.SW;
  xp.org = g.o - (n - 1);  // window of output block t: input rows from t·n + o − (n−1)
  set_xspec_tma(xp, B, 2 * n - 1);
  oaa::WalkParams wp{};
  wp.S = xp.S;
  wp.spec = spec;
  wp.out = y;
  wp.B = B;
  wp.Cin = C;
  wp.Cout = K;
  wp.T = o.Td;
  wp.Ro = g.M;
  wp.off = 0;
  wp.NCH = o.NCH;
  wp.KG = o.KG;
  wp.ngrp = o.ngrp;
  cudaError_t err = launch_walk_oas(n, xp, wp, o, C, s);
  prof.stop();
  return err == cudaSuccess ? OAA_OK : OAA_ERR_CUDA;
}

oaa_status_t oaa_conv_bwd_data(const float* dy, const float* w, float* dx, int B, int C, int K,
                               int N, int n, oaa_crop_t crop, void* ws, size_t ws_bytes,
                               void* stream) {
  return run_engine(false, dy, w, dx, B, C, K, N, n, crop, ws, ws_bytes, stream);
}

oaa_status_t oaa_conv_bwd_filter(const float* x, const float* dy, float* dw, int B, int C, int K,
                                 int N, int n, oaa_crop_t crop, void* ws, size_t ws_bytes,
                                 void* stream) {
  Geo g;
  oaa_status_t st = validate(B, C, K, N, n, crop, &g);
  if (st != OAA_OK) return st;
  if (!dw || (B > 0 && (!x || !dy))) return OAA_ERR_INVALID_VALUE;
  const size_t x_bytes = sizeof(float) * (size_t)B * C * N * N;
  const size_t dy_bytes = sizeof(float) * (size_t)B * K * g.M * g.M;
  const size_t dw_bytes = sizeof(float) * (size_t)K * C * n * n;
  if (overlaps(dw, dw_bytes, x, x_bytes) || overlaps(dw, dw_bytes, dy, dy_bytes))
    return OAA_ERR_INVALID_VALUE;
  // the documented v1 limit (include/oaa.h): max(ceil(N/n)·n, M) ≤ 256, as for the forward
  if (std::max(cdiv(N, n) * n, g.M) > oaa::kMaxThreads) return OAA_ERR_UNSUPPORTED;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (B == 0) {
    if (cudaMemsetAsync(dw, 0, dw_bytes, s) != cudaSuccess) return OAA_ERR_CUDA;
    return OAA_OK;
  }
  const TcFiltPlan tcf = plan_tc_filter(B, C, K, N, g.M, n);
  if (tcf.use) return run_filter_tc(x, dy, dw, B, C, K, N, n, g, tcf, ws, ws_bytes, s, x_bytes, dy_bytes, dw_bytes);
  const BwdfPlan bf = plan_bwdf(B, C, K, g.M, n);
  if (bf.use) {
    const size_t need = bf.xs_b + bf.part_b;
    if (!ws || ws_bytes < need || (reinterpret_cast<uintptr_t>(ws) % kAlign) != 0) return OAA_ERR_WORKSPACE;
    if (overlaps(ws, need, dw, dw_bytes) || overlaps(ws, need, x, x_bytes) || overlaps(ws, need, dy, dy_bytes))
      return OAA_ERR_INVALID_VALUE;
    char* base = static_cast<char*>(ws);
    oaa::XSpecParams xp;
    xp.in = x;
    xp.S = reinterpret_cast<float4*>(base);
    xp.Cin = C;
    xp.R = N;
    xp.T = bf.Td;
    xp.NCH = bf.NCH;
    xp.SW = bf.SW;
    xp.org = g.o - (n - 1);
    set_xspec_tma(xp, B, 2 * n - 1);
    oaa::BwdFParams fp;
    fp.dy = dy;
    fp.XS = xp.S;
    fp.partial = reinterpret_cast<float2*>(base + bf.xs_b);
    fp.B = B;
    fp.K = K;
    fp.C = C;
    fp.M = g.M;
    fp.Td = bf.Td;
    fp.NCH = bf.NCH;
    fp.G = bf.G;
    fp.KG = bf.KG;
    ProfScope prof(OAA_OP_BWD_FILTER, s);
    prof.start();
    cudaError_t err = launch_bwdf(n, xp, fp, BwdfLaunch{bf.xspec_smem, bf.smem, bf.nkg, bf.tm}, s);
    prof.stop();
    if (err != cudaSuccess) return OAA_ERR_CUDA;
    launch_finalize(fp.partial, dw, bf.G, K, C, n, s);
    g_launches++;
    return cudaGetLastError() == cudaSuccess ? OAA_OK : OAA_ERR_CUDA;
  }
  FilterPlan f;
  if (!plan_filter(B, C, K, g.M, n, &f)) return OAA_ERR_UNSUPPORTED;
  const size_t need = align_up(sizeof(float2) * (size_t)f.G * K * C * g.P * g.H);
  if (!ws || ws_bytes < need || (reinterpret_cast<uintptr_t>(ws) % kAlign) != 0)
    return OAA_ERR_WORKSPACE;
  if (overlaps(ws, need, dw, dw_bytes) || overlaps(ws, need, x, x_bytes) ||
      overlaps(ws, need, dy, dy_bytes))
    return OAA_ERR_INVALID_VALUE;
  oaa::FilterParams p;
  p.x = x;
  p.dy = dy;
  p.partial = static_cast<float2*>(ws);
  p.B = B;
  p.C = C;
  p.K = K;
  p.N = N;
  p.M = g.M;
  p.off = g.o;
  p.Td = f.Td;
  p.G = f.G;
  p.KG = f.KG;
  p.TCH = f.TCH;
  p.XW = f.XW;
  p.DW = f.DW;
  ProfScope prof(OAA_OP_BWD_FILTER, s);
  prof.start();
  cudaError_t err = launch_filter(n, p, f, s);
  prof.stop();
  if (err != cudaSuccess) return OAA_ERR_CUDA;
  launch_finalize(static_cast<const float2*>(ws), dw, f.G, K, C, n, s);
  g_launches++;
  if (cudaGetLastError() != cudaSuccess) return OAA_ERR_CUDA;
  return OAA_OK;
}

size_t oaa_weight_spectra_bytes(oaa_op_t op, int C, int K, int N, int n, oaa_crop_t crop) {
  Geo g;
  if (op != OAA_OP_FWD && op != OAA_OP_BWD_DATA) return 0;
  if (validate(1, C, K, N, n, crop, &g) != OAA_OK) return 0;
  const SpecPlan sp = spec_plan(op == OAA_OP_FWD, C, K, N, n, g);
  return sp.ok ? sp.bytes : 0;
}

oaa_status_t oaa_weight_spectra(oaa_op_t op, const float* w, void* spec, size_t spec_bytes, int C, int K, int N,
                                int n, oaa_crop_t crop, void* stream) {
  Geo g;
  if (op != OAA_OP_FWD && op != OAA_OP_BWD_DATA) return OAA_ERR_INVALID_VALUE;
  oaa_status_t st = validate(1, C, K, N, n, crop, &g);
  if (st != OAA_OK) return st;
  if (!w || !spec || (reinterpret_cast<uintptr_t>(spec) % kAlign) != 0) return OAA_ERR_INVALID_VALUE;
  const bool is_fwd = op == OAA_OP_FWD;
  const SpecPlan sp = spec_plan(is_fwd, C, K, N, n, g);
  if (!sp.ok) return OAA_ERR_UNSUPPORTED;
  if (spec_bytes < sp.bytes) return OAA_ERR_WORKSPACE;
  if (overlaps(spec, sp.bytes, w, sizeof(float) * (size_t)K * C * n * n)) return OAA_ERR_INVALID_VALUE;
  // run the call's own spectrum stage into `spec`: a B = 1 call with the spectra as its
  // workspace prefix would also launch the main kernels, so the stage is issued directly
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int R = is_fwd ? N : g.M, Ro = is_fwd ? g.M : N;
  const int Cin = is_fwd ? C : K, Cout = is_fwd ? K : C;
  const int off = is_fwd ? g.o : (n - 1 - g.o);
  const TcPlan tc = plan_tc(1, Cin, Cout, R, n);
  KTimer kt(KID_SPECTRUM, s);
  if (tc.use) {
    if (cudaMemsetAsync(spec, 0, tc.ag_b, s) != cudaSuccess) return OAA_ERR_CUDA;
    const long long total = (long long)tc.F * Cin * Cout;
    const int blocks = (int)std::min<long long>((total + 255) / 256, 8192);
    oaa::oaa_realified_spectrum_kernel<<<blocks, 256, 0, s>>>(w, static_cast<float*>(spec), K, C, n, tc.P, is_fwd ? 0 : 1,
                                                              tc.Kc, tc.RTA);
  } else {
    EnginePlan e;
    plan_engine(R, Ro, off, n, Cin, Cout, &e, false);
    const WalkHostGeo wk = plan_walk(is_fwd, 1, Cin, Cout, R, Ro, off, n, tc);
    const BwddPlan bd = plan_bwdd(is_fwd, 1, Cout, R, n, tc);
    const int loop_is_k = (wk.use || bd.use) ? 1 : ((is_fwd == e.S1) ? 1 : 0);
    oaa::oaa_spectrum_kernel<<<K * C, 128, 0, s>>>(w, static_cast<float4*>(spec), K, C, n, wk.use ? wk.P : bd.use ? bd.P : 2 * n - 1, is_fwd ? 0 : 1,
                                                    loop_is_k);
  }
  g_launches++;
  return cudaGetLastError() == cudaSuccess ? OAA_OK : OAA_ERR_CUDA;
}

oaa_status_t oaa_conv_fwd_prepared(const float* x, const void* spec, float* y, int B, int C, int K, int N, int n,
                                   oaa_crop_t crop, void* ws, size_t ws_bytes, void* stream) {
  if (!spec) return OAA_ERR_INVALID_VALUE;
  return run_engine(true, x, nullptr, y, B, C, K, N, n, crop, ws, ws_bytes, stream, spec);
}

oaa_status_t oaa_conv_bwd_data_prepared(const float* dy, const void* spec, float* dx, int B, int C, int K, int N,
                                        int n, oaa_crop_t crop, void* ws, size_t ws_bytes, void* stream) {
  if (!spec) return OAA_ERR_INVALID_VALUE;
  return run_engine(false, dy, nullptr, dx, B, C, K, N, n, crop, ws, ws_bytes, stream, spec);
}

const char* oaa_status_string(oaa_status_t s) {
  switch (s) {
    case OAA_OK: return "OAA_OK";
    case OAA_ERR_INVALID_VALUE: return "OAA_ERR_INVALID_VALUE: invalid argument";
    case OAA_ERR_UNSUPPORTED: return "OAA_ERR_UNSUPPORTED: size outside v1 limits (n<=8, N<=~250)";
    case OAA_ERR_WORKSPACE: return "OAA_ERR_WORKSPACE: workspace too small or misaligned";
    case OAA_ERR_CUDA: return "OAA_ERR_CUDA: CUDA launch failure";
  }
  return "unknown oaa_status_t";
}

size_t oaa_debug_bin_gemm_workspace_bytes(int F, int M, int N, int Kd) {
  if (F < 1 || M < 1 || N < 1 || Kd < 1) return 0;
  const size_t NB = N > oaa::kTcM ? 2 : 1;
  const size_t Kc = cdiv(Kd, oaa::kTcK), RTA = cdiv(M, oaa::kTcM), RTB = (cdiv(cdiv(N, oaa::kTcM), (int)NB)) * NB;
  return align_up(sizeof(float) * (size_t)F * Kc * RTA * 4096) + align_up(sizeof(float) * (size_t)F * Kc * RTB * 4096);
}

oaa_status_t oaa_debug_bin_gemm(const float* A, const float* B, float* D, int F, int M, int N, int Kd, void* ws,
                                size_t ws_bytes, void* stream) {
  if (!A || !B || !D || F < 1 || M < 1 || N < 1 || Kd < 1) return OAA_ERR_INVALID_VALUE;
  const size_t need = oaa_debug_bin_gemm_workspace_bytes(F, M, N, Kd);
  if (!ws || ws_bytes < need || (reinterpret_cast<uintptr_t>(ws) % kAlign) != 0) return OAA_ERR_WORKSPACE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  oaa::BinGemmParams p{};
  p.F = F; p.M = M; p.N = N; p.ldd = N;
  p.NB = N > oaa::kTcM ? 2 : 1;
  p.Kc = cdiv(Kd, oaa::kTcK); p.RTA = cdiv(M, oaa::kTcM); p.RTB = cdiv(cdiv(N, oaa::kTcM), p.NB) * p.NB;
  p.strideD = (long long)M * N;
  p.S = 1; p.kps = p.Kc; p.mode = 0; p.partial = nullptr; p.accumulate = 0; p.Kuse = p.Kc;
  float* Ap = static_cast<float*>(ws);
  float* Bp = reinterpret_cast<float*>(static_cast<char*>(ws) + align_up(sizeof(float) * (size_t)F * p.Kc * p.RTA * 4096));
  oaa::oaa_tc_pack_kernel<<<1024, 256, 0, s>>>(A, Ap, F, M, Kd, p.Kc, p.RTA);
  g_launches++;
  oaa::oaa_tc_pack_kernel<<<1024, 256, 0, s>>>(B, Bp, F, N, Kd, p.Kc, p.RTB);
  g_launches++;
  if (cudaGetLastError() != cudaSuccess) return OAA_ERR_CUDA;
  p.A = Ap; p.B = Bp; p.D = D;
  return launch_bin_gemm(p, s) == cudaSuccess ? OAA_OK : OAA_ERR_CUDA;
}

static const char* const kKernelNames[KID_COUNT] = {
    "spectrum", "xspec", "walk", "bwdd", "xspec_win", "bwdf", "finalize",
    "tile_spectra", "bin_gemm", "walk_load", "filter_spectra", "engine", "aux", "walk_oas", "bwd_fused"};

int oaa_profile_kernel_count(void) { return KID_COUNT; }

const char* oaa_profile_kernel_name(int id) { return (id >= 0 && id < KID_COUNT) ? kKernelNames[id] : nullptr; }

int oaa_profile_collect_kernels(double* ms, int* count, int n) {
  std::vector<KRec> recs;
  {
    std::lock_guard<std::mutex> g(g_prof_mu);
    recs.swap(g_kprof);
  }
  for (int i = 0; i < n; ++i) {
    if (ms) ms[i] = 0.0;
    if (count) count[i] = 0;
  }
  int bad = 0;
  for (auto& r : recs) {
    if (cudaEventSynchronize(r.b) != cudaSuccess) bad = 1;
    float t = 0.f;
    if (cudaEventElapsedTime(&t, r.a, r.b) != cudaSuccess) bad = 1;
    if (r.kid >= 0 && r.kid < n) {
      if (ms) ms[r.kid] += t;
      if (count) count[r.kid] += 1;
    }
  }
  {
    std::lock_guard<std::mutex> g(g_prof_mu);
    for (auto& r : recs) {
      g_event_pool.push_back(r.a);
      g_event_pool.push_back(r.b);
    }
  }
  return bad ? -1 : (int)recs.size();
}

const char* oaa_version(void) { return "oaa-b200 0.1.0 sm_100a"; }

int oaa_block_size(oaa_op_t op, int C, int K, int N, int n, oaa_crop_t crop) {
  Geo g;
  if (op != OAA_OP_FWD && op != OAA_OP_BWD_DATA) return -1;
  if (validate(1, C, K, N, n, crop, &g) != OAA_OK) return -1;
  const bool fwd = op == OAA_OP_FWD;
  const int R = fwd ? N : g.M, Ro = fwd ? g.M : N, off = fwd ? g.o : (n - 1 - g.o);
  const int Cin = fwd ? C : K, Cout = fwd ? K : C;
  const TcPlan tc = plan_tc(1, Cin, Cout, R, n);
  if (tc.use) return tc.BB;
  const WalkHostGeo wk = plan_walk(fwd, 1, Cin, Cout, R, Ro, off, n, tc);
  if (wk.use) return wk.BB;
  const BwddPlan bd = plan_bwdd(fwd, 1, Cout, R, n, tc);
  return bd.use ? bd.BB : n;
}

uint64_t oaa_launch_count(void) { return g_launches.load(); }

void oaa_profile_enable(int on) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  g_prof_on = on != 0;
}

int oaa_profile_collect(double* ms, int* count) {
  std::vector<ProfRec> recs;
  {
    std::lock_guard<std::mutex> g(g_prof_mu);
    recs.swap(g_prof);
  }
  for (int i = 0; i < 3; ++i) {
    if (ms) ms[i] = 0.0;
    if (count) count[i] = 0;
  }
  int bad = 0;
  for (auto& r : recs) {
    if (cudaEventSynchronize(r.b) != cudaSuccess) bad = 1;
    float t = 0.f;
    if (cudaEventElapsedTime(&t, r.a, r.b) != cudaSuccess) bad = 1;
    if (r.op >= 0 && r.op < 3) {
      if (ms) ms[r.op] += t;
      if (count) count[r.op] += 1;
    }
  }
  {
    std::lock_guard<std::mutex> g(g_prof_mu);
    for (auto& r : recs) {
      g_event_pool.push_back(r.a);
      g_event_pool.push_back(r.b);
    }
  }
  return bad ? -1 : (int)recs.size();
}

}  // extern "C"
