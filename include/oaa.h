/*
 * oaa.h -- C ABI of liboaa.so, the B200 (sm_100a) overlap-and-add convolution layer of
 * Highlander & Rodriguez, "Very Efficient Training of Convolutional Neural Networks
 * using Fast Fourier Transform and Overlap-and-Add" (arXiv 1601.06815).
 *
 * The operations (citations are /root/reference/PAPER.md lines; SPEC.md lines are the
 * spec written from the paper):
 *
 *   oaa_conv_fwd        the convolutional layer's forward propagation: K output maps,
 *                       each the sum over the C input channels of the channel convolved
 *                       with the matching kernel channel (§1 "The total
 *                       number of convolutions in a CNN convolutional layer is KC"),
 *                       computed by overlap-and-add (§2: the N×N input is
 *                       broken into ceil(N/n)² n×n blocks, each block convolution is a
 *                       Hadamard product in the frequency domain on a (2n−1)-point grid
 *                       (PAPER.md:27, :85), and the results are "overlapped by n−1 ...
 *                       and added together").  True convolution (kernel flipped;
 *                       SPEC.md:267).
 *   oaa_conv_bwd_data   "one convolution to propagate the error through the layer"
 *                       (§3.2): dx = Σ_k FullConv(dy_k, flip180 w_kc),
 *                       cropped at offset n−1−o (the adjoint of the forward).
 *   oaa_conv_bwd_filter "another to calculate the change in weight":
 *                       dw[k,c,u,v] = Σ_b Σ_a x[b,c,a]·G[b,k,a+(u,v)], G = dy placed at
 *                       offset o in the (N+n−1)² Full frame (the adjoint w.r.t. w).
 *
 * Shapes and layouts (all dense, row-major, fp32, DEVICE memory):
 *   x, dx : [B][C][N][N]      w, dw : [K][C][n][n]      y, dy : [B][K][M][M]
 *   crop  : OAA_CROP_FULL  M = N+n−1, o = 0
 *           OAA_CROP_VALID M = N−n+1, o = n−1   (requires n ≤ N)
 *           OAA_CROP_SAME  M = N,     o = floor((n−1)/2)  (= scipy 'same')
 *   (Valid is the layer default.)  Stride 1, no dilation,
 *   no bias (readings R5, R6, R12).
 *
 * Supported sizes (v1): 1 ≤ n ≤ 8; max(ceil(R/n)·n, Ro) ≤ 256 where (R, Ro) is
 * (N, M) for fwd and bwd_filter and (M, N) for bwd_data (i.e. N up to ≈ 250);
 * B, C, K ≥ 1 (B = 0 is a no-op; bwd_filter then zero-fills dw).  Anything else returns
 * OAA_ERR_UNSUPPORTED (size limits) or OAA_ERR_INVALID_VALUE (nonsense arguments)
 * and writes nothing.
 *
 * Ownership / threading: the caller owns every buffer including the workspace (size
 * from oaa_conv_workspace_bytes; ≥ 256-byte aligned).  The library never allocates,
 * frees or synchronises; every call enqueues kernels on `stream` (a cudaStream_t,
 * NULL = legacy default stream) and returns immediately -- results are valid in stream
 * order.  Outputs are fully overwritten, never accumulated; dw is the sum over this
 * call's B images only (the cross-GPU sum is the caller's all-reduce).  Concurrent
 * calls must use distinct workspaces.  Results are bitwise deterministic for a given
 * device and arguments (bwd_data adds the two overlapping contributions of a dx element
 * with red.add onto an exact zero, which is order-independent).  Internally the kernels
 * allocate tensor memory (tcgen05.alloc, ≤ 512 columns per SM) for their accumulators and
 * release it before they exit.
 *
 * Errors: arguments are validated on the host before any launch; on error nothing is
 * written.  Launch failures are reported as OAA_ERR_CUDA (the call stays asynchronous).
 */
#ifndef OAA_H_
#define OAA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
/* liboaa.so is built with hidden default visibility: exactly the declarations below are
   exported. */
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

typedef enum { OAA_CROP_FULL = 0, OAA_CROP_VALID = 1, OAA_CROP_SAME = 2 } oaa_crop_t;

typedef enum {
  OAA_OK = 0,
  OAA_ERR_INVALID_VALUE = 1, /* null pointer, negative size, bad crop, Valid with n > N, aliasing */
  OAA_ERR_UNSUPPORTED = 2,   /* valid arguments outside the v1 size limits */
  OAA_ERR_WORKSPACE = 3,     /* ws_bytes < oaa_conv_workspace_bytes(...) or ws misaligned */
  OAA_ERR_CUDA = 4           /* a kernel launch or memset failed (cudaGetLastError) */
} oaa_status_t;

typedef enum {
  OAA_OP_FWD = 0,
  OAA_OP_BWD_DATA = 1,
  OAA_OP_BWD_FILTER = 2,
  OAA_OP_FWD_OAS = 3, /* oaa_conv_fwd_oas */
  OAA_OP_BWD = 4      /* oaa_conv_bwd (fused backward) */
} oaa_op_t;

/* Output side M for input side N and kernel side n; −1 if invalid. */
int oaa_conv_out_size(int N, int n, oaa_crop_t crop);

/* Workspace bytes needed by `op` for these arguments (0 is a valid answer only for
 * B = 0).  Depends only on the arguments.  Returns 0 for invalid arguments. */
size_t oaa_conv_workspace_bytes(oaa_op_t op, int B, int C, int K, int N, int n, oaa_crop_t crop);

/* y[B][K][M][M] = crop(Σ_c x[b,c] ∗ w[k,c]).  x, w, y: device pointers. */
oaa_status_t oaa_conv_fwd(const float* x, const float* w, float* y, int B, int C, int K, int N,
                          int n, oaa_crop_t crop, void* ws, size_t ws_bytes, void* stream);

/* The same y as oaa_conv_fwd, computed by OVERLAP-AND-SAVE (§1: "the
 * overlap-and-save ... is a similar technique that may be marginally faster but has the same
 * complexity").  Output block t (n×n, at t·n in the cropped
 * output) is the last n rows and columns of the P-point CIRCULAR convolution (P = 2n−1)
 * of the kernel with the (2n−1)² input window starting at t·n + o − (n−1) (zero outside
 * x): those outputs have no wrap-around, so they equal the linear convolution and every
 * output is written once, with no overlap-add.  Workspace: op OAA_OP_FWD_OAS.  Supported
 * for C ≤ 4 (the SIMT walker family: window spectra, then the walker in overlap-and-save mode)
 * and for C, K ≥ 16 (the tensor-core path: window spectra of the output tiles, tcgen05 bin
 * GEMM, walker in load + overlap-and-save mode); other channel counts return
 * OAA_ERR_UNSUPPORTED.  Other arguments, layouts, limits and errors as oaa_conv_fwd. */
oaa_status_t oaa_conv_fwd_oas(const float* x, const float* w, float* y, int B, int C, int K, int N,
                              int n, oaa_crop_t crop, void* ws, size_t ws_bytes, void* stream);

/* dx[B][C][N][N] from dy[B][K][M][M] and w.  dy, w, dx: device pointers. */
oaa_status_t oaa_conv_bwd_data(const float* dy, const float* w, float* dx, int B, int C, int K,
                               int N, int n, oaa_crop_t crop, void* ws, size_t ws_bytes,
                               void* stream);

/* dw[K][C][n][n] = Σ over this call's batch.  x, dy, dw: device pointers. */
oaa_status_t oaa_conv_bwd_filter(const float* x, const float* dy, float* dw, int B, int C, int K,
                                 int N, int n, oaa_crop_t crop, void* ws, size_t ws_bytes,
                                 void* stream);

/* Prepared (cached) weight spectra -- SURVEY.md §8(f) NEXT-4, SPEC.md:266 ("a caller-
 * visible 'prepared kernel' cache ... for layer-level reuse across many inputs").  Every
 * fwd / bwd_data call first transforms the kernels (a1: Ŵ = DFT_P(w), or of flip180(w)
 * for bwd_data) into its workspace; with fixed weights (inference, or many calls per
 * optimizer step) that stage can be done once:
 *   bytes = oaa_weight_spectra_bytes(op, C, K, N, n, crop);       op: FWD or BWD_DATA
 *   oaa_weight_spectra(op, w, spec, bytes, C, K, N, n, crop, stream);
 *   oaa_conv_fwd_prepared(x, spec, y, B, C, K, N, n, crop, ws, ws_bytes, stream);  (×many)
 * The layout is internal (it depends on which kernel family the arguments select) and
 * is valid only for the same (op, C, K, N, n, crop); results are bitwise those of the
 * unprepared call.  spec: caller-owned device buffer, 256-byte aligned, never written
 * by the *_prepared calls; the caller re-prepares after changing w.  Workspace sizes as
 * for the unprepared op.  Errors as for the conv calls (OAA_ERR_WORKSPACE if spec_bytes
 * is too small; op other than FWD / BWD_DATA is OAA_ERR_INVALID_VALUE). */
size_t oaa_weight_spectra_bytes(oaa_op_t op, int C, int K, int N, int n, oaa_crop_t crop);
oaa_status_t oaa_weight_spectra(oaa_op_t op, const float* w, void* spec, size_t spec_bytes, int C, int K, int N,
                                int n, oaa_crop_t crop, void* stream);
oaa_status_t oaa_conv_fwd_prepared(const float* x, const void* spec, float* y, int B, int C, int K, int N, int n,
                                   oaa_crop_t crop, void* ws, size_t ws_bytes, void* stream);
oaa_status_t oaa_conv_bwd_data_prepared(const float* dy, const void* spec, float* dx, int B, int C, int K, int N,
                                        int n, oaa_crop_t crop, void* ws, size_t ws_bytes, void* stream);

/* The whole backward pass in one call (§3.2: "the backward propagation
 * contains two actual convolutions per kernel: one convolution to propagate the error
 * through the layer and another to calculate the change in weight"; SURVEY.md §8(f)
 * NEXT-1): dx as oaa_conv_bwd_data(dy, w) and dw as oaa_conv_bwd_filter(x, dy), both
 * written.  On the tensor-core path (C, K ≥ 16) the dy blocks are read and transformed
 * ONCE per batch chunk: the same spectra Ĝ feed the data-gradient contraction (Σ over
 * k) and the weight-gradient accumulation (Σ over blocks).  Elsewhere the two
 * convolutions run back to back on `stream`.  dw may differ from a separate
 * oaa_conv_bwd_filter call in rounding (the fused path's batch chunks set its split-K
 * order); results are deterministic for given arguments.  Workspace: op OAA_OP_BWD.
 * Arguments, layouts, limits and errors as the two separate calls; all of x, dy, w, dx,
 * dw and ws must be pairwise disjoint. */
oaa_status_t oaa_conv_bwd(const float* x, const float* dy, const float* w, float* dx, float* dw, int B, int C,
                          int K, int N, int n, oaa_crop_t crop, void* ws, size_t ws_bytes, void* stream);

/* Diagnostic entry point of the tensor-core contraction used for large C·K (SURVEY.md
 * §8(a) a4): D[f] = A[f]·B[f]ᵀ for f < F, A[f] M×Kd, B[f] N×Kd, D[f] M×N, all row-major
 * fp32 device arrays, evaluated with tcgen05 3×TF32 (fp32-accurate).  The operands are
 * first packed (plain fp32, UMMA-blocked) into the caller's workspace of
 * oaa_debug_bin_gemm_workspace_bytes(F, M, N, Kd) bytes; the kernel's converter warps
 * split them into TF32 hi/lo in shared memory.  Exposed so tests can check the
 * tensor-core kernel in isolation. */
size_t oaa_debug_bin_gemm_workspace_bytes(int F, int M, int N, int Kd);
oaa_status_t oaa_debug_bin_gemm(const float* A, const float* B, float* D, int F, int M, int N, int Kd,
                                void* ws, size_t ws_bytes, void* stream);

/* Block size b the call (op = FWD or BWD_DATA) with these arguments tiles its input into
 * (host-side planning only, no GPU work): n for the paper's OaA (blocks of the
 * kernel's size), 16 − n when the forward walker / bwd_data kernels (C ≤ 4 input / output
 * channels) or the tensor-core path (C, K ≥ 16) use larger blocks on the P = b + n − 1 = 15
 * grid (R18).  Returns −1 for invalid arguments or another
 * op. */
int oaa_block_size(oaa_op_t op, int C, int K, int N, int n, oaa_crop_t crop);

/* Static description of a status code. */
const char* oaa_status_string(oaa_status_t s);

/* Library version string ("oaa-b200 <semver> sm_100a"). */
const char* oaa_version(void);

/* Number of kernels this process has launched through the library so far (monotone;
 * used by bench.py to report gpu_launches). */
uint64_t oaa_launch_count(void);

/* Kernel timing for the roofline report.  When enabled, every call records CUDA events
 * around its main (dominant) kernel on the call's stream; oaa_profile_collect
 * synchronises those events, writes the summed milliseconds and launch counts per op
 * (index = oaa_op_t) into ms[3] / count[3], and clears the record.  Returns the
 * number of records collected or −1 on a CUDA error. */
void oaa_profile_enable(int on);
int oaa_profile_collect(double* ms, int* count);

/* Per-kernel timing (same enable switch): every launch records CUDA events on its
 * stream, labelled with a kernel id in [0, oaa_profile_kernel_count()).
 * oaa_profile_collect_kernels synchronises them, writes the summed milliseconds and
 * launch counts of the first n ids into ms[n] / count[n] (either may be NULL), clears
 * the record and returns the number of launches collected (−1 on a CUDA error).
 * oaa_profile_kernel_name(id) is a static name ("walk", "bwdd", "bin_gemm", ...), NULL
 * for an unknown id. */
int oaa_profile_kernel_count(void);
const char* oaa_profile_kernel_name(int id);
int oaa_profile_collect_kernels(double* ms, int* count, int n);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif
#endif /* OAA_H_ */
