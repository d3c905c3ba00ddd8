"""Independent CPU float64 references that follow the paper's algorithms step by step.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Shares nothing with the CUDA path.

* ``oaa_conv_fwd`` -- overlap-and-add convolution exactly in the paper's order
  (§2 "the input is broken into N²/n² (rounded up) blocks equal to the
  kernel size n×n. A convolution between each block and the kernel is computed and the
  results are overlapped and added"; PAPER.md:27 each block convolution "in the
  frequency domain"; §3.2 zero-padded "so that each side is ... 2n−1 in
  OaAconv"; PAPER.md:15 the K·C convolutions of a layer):

    1. partition each N×N channel into ceil(N/n)² n×n blocks, zero-filling edge blocks
       (reading R1/R13);
    2. zero-pad each block and each kernel (top-left anchored) to P×P, P ≥ 2n−1
       (default P = 2n−1, reading R3);
    3. forward DFT of every padded block and kernel (unnormalised; reading R10);
    4. Hadamard product with the kernel spectrum, summed over the C channels for each
       of the K kernels (sum-before-inverse is reading R8);
    5. inverse DFT with 1/P²; keep the real part;
    6. overlap-add block (t1, t2) at (t1·n, t2·n) into a (T·n+n−1)² accumulator
       (the n−1 overlap of PAPER.md:18; SPEC.md:78 accumulate_at);
    7. crop to Full / Valid / Same (reading R5).

  The DFT is the plain definition written as a matrix (``dft_matrix``), valid for any
  P; ``use_numpy_fft=True`` swaps in numpy's FFT library primitive instead.  An optional
  block size ``b`` (default n, the paper's) partitions into b×b blocks, overlap-added at
  stride b, at P = b + n − 1 -- the product's b ≠ n blocks (reading R18).

* ``oaa_conv_bwd_data`` / ``oaa_conv_bwd_filter`` -- the same OaA machinery applied to
  the two backward convolutions of PAPER.md:89 (reading R7): bwd_data is OaA of dy with
  the flipped kernels, cropped at n−1−o; bwd_filter correlates dy n×n blocks with the
  (2n−1)² x-windows that overlap them, sums the products in frequency, inverse
  transforms and reads the lags (n−1−u, n−1−v).

* ``oas_conv_fwd`` -- overlap-and-save (textbook segments + circular
  convolution + discarded aliased samples), the reference for the OaS forward variant.

* ``fft_conv_fwd`` -- "FFTconv", whole-array Hadamard product at next_pow2(N+n−1)
  (SPEC.md:211-214), the third independent implementation.

Shapes may be rectangular ([.., rows, cols]); kernels are always smaller-or-equal
rectangular blocks.
"""
from __future__ import annotations

import math

import numpy as np

CROP = {"full": 0, "valid": 1, "same": 2}


# ----------------------------------------------------------------------------- shapes
def out_size(N: int, n: int, crop) -> int:
    """SPEC.md:188 ConvMode sizes."""
    c = CROP[crop] if isinstance(crop, str) else int(crop)
    if c == 0:
        return N + n - 1
    if c == 1:
        if n > N:
            raise ValueError("Valid mode requires n <= N (SPEC.md:206)")
        return N - n + 1
    if c == 2:
        return N
    raise ValueError(crop)


def crop_offset(n: int, crop) -> int:
    """Full 0, Valid n−1, Same floor((n−1)/2)."""
    c = CROP[crop] if isinstance(crop, str) else int(crop)
    return {0: 0, 1: n - 1, 2: (n - 1) // 2}[c]


def next_pow2(m: int) -> int:
    """SPEC.md:112."""
    if m < 1:
        raise ValueError("next_pow2 of m < 1")
    p = 1
    while p < m:
        p *= 2
    return p


# ------------------------------------------------------------------------------- DFT
def dft_matrix(P: int, sign: int = -1) -> np.ndarray:
    """F[f, p] = exp(sign·2πi·f·p/P)  (the DFT definition)."""
    f = np.arange(P).reshape(P, 1)
    p = np.arange(P).reshape(1, P)
    return np.exp(sign * 2j * np.pi * ((f * p) % P) / P)


def dft2(a: np.ndarray, P1: int, P2: int | None = None, use_numpy_fft: bool = False) -> np.ndarray:
    """Unnormalised forward 2-D DFT of the last two axes of ``a`` zero-padded
    (top-left anchored) to P1×P2.  Row-column (separable) evaluation of
    the definition X[f1,f2] = Σ_p a[p1,p2] e^{−2πi(f1p1/P1 + f2p2/P2)}."""
    P2 = P1 if P2 is None else P2
    r, c = a.shape[-2:]
    if r > P1 or c > P2:
        raise ValueError("zero_pad: target smaller than input (SPEC.md:55)")
    pad = np.zeros(a.shape[:-2] + (P1, P2), dtype=np.complex128)
    pad[..., :r, :c] = a
    if use_numpy_fft:
        return np.fft.fft2(pad, axes=(-2, -1))
    F1 = dft_matrix(P1, -1)
    F2 = dft_matrix(P2, -1)
    return np.einsum("fp,...pq,gq->...fg", F1, pad, F2)


def idft2(A: np.ndarray, use_numpy_fft: bool = False) -> np.ndarray:
    """Inverse 2-D DFT with the 1/(P1·P2) normalisation."""
    P1, P2 = A.shape[-2:]
    if use_numpy_fft:
        return np.fft.ifft2(A, axes=(-2, -1))
    G1 = dft_matrix(P1, +1)
    G2 = dft_matrix(P2, +1)
    return np.einsum("pf,...fg,qg->...pq", G1, A, G2) / (P1 * P2)


# ------------------------------------------------------------------ block partition
def partition_blocks(a: np.ndarray, nr: int, nc: int | None = None):
    """Split the last two axes into ceil(N/n) × ceil(N/n) non-overlapping n×n blocks,
    zero-filling the edge blocks ("rounded up").

    Returns (blocks[..., T1, T2, nr, nc], origins list of (row, col)).
    """
    nc = nr if nc is None else nc
    R, Cc = a.shape[-2:]
    T1, T2 = -(-R // nr), -(-Cc // nc)
    pad = np.zeros(a.shape[:-2] + (T1 * nr, T2 * nc), dtype=a.dtype)
    pad[..., :R, :Cc] = a
    blocks = pad.reshape(a.shape[:-2] + (T1, nr, T2, nc))
    blocks = np.moveaxis(blocks, -3, -2)  # [..., T1, T2, nr, nc]
    origins = [(t1 * nr, t2 * nc) for t1 in range(T1) for t2 in range(T2)]
    return blocks, origins


def _crop(full: np.ndarray, N_r: int, N_c: int, n_r: int, n_c: int, crop) -> np.ndarray:
    Mr, Mc = out_size(N_r, n_r, crop), out_size(N_c, n_c, crop)
    orr, oc = crop_offset(n_r, crop), crop_offset(n_c, crop)
    return full[..., orr:orr + Mr, oc:oc + Mc]


# --------------------------------------------------------------------- OaA forward
def _oaa_full(x: np.ndarray, w: np.ndarray, P1: int, P2: int, use_numpy_fft: bool,
              return_imag: bool = False, b=None):
    """Steps 1-6: the Full (N+n−1) linear convolution by overlap-and-add.
    x[B,C,R,Cc], w[K,C,nr,nc] -> Full[B,K,R+nr−1,Cc+nc−1].
    b: block size (default the kernel's, as in the paper); any b gives the same
    linear convolution when P ≥ b + n − 1 (reading R18, the product's b ≠ n blocks)."""
    B, C, R, Cc = x.shape
    K, C2, nr, nc = w.shape
    assert C == C2
    br, bc = (nr, nc) if b is None else ((b, b) if np.isscalar(b) else b)
    if P1 < br + nr - 1 or P2 < bc + nc - 1:
        # Not an error for the reference: it lets tests show aliasing when P < b+n−1.
        pass
    blocks, _ = partition_blocks(x.astype(np.float64), br, bc)        # step 1
    T1, T2 = blocks.shape[2], blocks.shape[3]
    Xh = dft2(blocks, P1, P2, use_numpy_fft)                          # steps 2-3: [B,C,T1,T2,P1,P2]
    Wh = dft2(w.astype(np.float64), P1, P2, use_numpy_fft)            # kernel spectrum once
    Yh = np.einsum("kcfg,bcstfg->bkstfg", Wh, Xh)                     # step 4: Hadamard, Σ_c
    yb = idft2(Yh, use_numpy_fft)                                     # step 5
    imag = np.abs(yb.imag).max() if yb.size else 0.0
    yb = yb.real
    # Each block result is the (b+n−1)-sized linear conv of a b×b block with an n×n
    # kernel; entries beyond b+n−1 are zero when P ≥ b+n−1 (or aliased when not).
    Lr, Lc = min(P1, br + nr - 1), min(P2, bc + nc - 1)
    full = np.zeros((B, K, T1 * br + nr - 1, T2 * bc + nc - 1))
    for t1 in range(T1):                                              # step 6: overlap-add
        for t2 in range(T2):
            full[:, :, t1 * br:t1 * br + Lr, t2 * bc:t2 * bc + Lc] += yb[:, :, t1, t2, :Lr, :Lc]
    full = full[:, :, :R + nr - 1, :Cc + nc - 1]
    return (full, imag) if return_imag else full


def _grid(n_r, n_c, P, b):
    """P per axis: given, else b + n − 1 (b = n: the paper's 2n − 1)."""
    br, bc = (n_r, n_c) if b is None else ((b, b) if np.isscalar(b) else b)
    P1 = br + n_r - 1 if P is None else (P if np.isscalar(P) else P[0])
    P2 = bc + n_c - 1 if P is None else (P if np.isscalar(P) else P[1])
    return P1, P2


def oaa_conv_fwd(x, w, crop="valid", P=None, use_numpy_fft=False, return_imag=False, b=None):
    """y = crop(OaA(x, w)) in float64.  x[B,C,R,Cc], w[K,C,nr,nc]; b: block size (R18)."""
    nr, nc = w.shape[-2:]
    P1, P2 = _grid(nr, nc, P, b)
    full, imag = _oaa_full(np.asarray(x), np.asarray(w), P1, P2, use_numpy_fft, True, b)
    y = _crop(full, x.shape[-2], x.shape[-1], nr, nc, crop)           # step 7
    return (y, imag) if return_imag else y


# ------------------------------------------------------------------- OaA bwd_data
def oaa_conv_bwd_data(dy, w, N, crop="valid", P=None, use_numpy_fft=False, b=None):
    """dx = crop_{[n−1−o, n−1−o+N)}( Σ_k FullConv(dy_k, flip180 w_{k,c}) ), the
    convolution "to propagate the error", itself computed by OaA on
    dy tiles with the flipped, transposed kernel set (reading R7).  N may be an
    int (square) or a (rows, cols) pair."""
    dy = np.asarray(dy, dtype=np.float64)
    w = np.asarray(w, dtype=np.float64)
    Nr, Nc = (N, N) if np.isscalar(N) else N
    nr, nc = w.shape[-2:]
    wflip = w[:, :, ::-1, ::-1].transpose(1, 0, 2, 3)                 # [C,K,nr,nc]
    P1, P2 = _grid(nr, nc, P, b)
    full = _oaa_full(dy, wflip, P1, P2, use_numpy_fft, False, b)      # [B,C,Mr+nr−1,Mc+nc−1]
    sr = nr - 1 - crop_offset(nr, crop)
    sc = nc - 1 - crop_offset(nc, crop)
    return full[:, :, sr:sr + Nr, sc:sc + Nc]


# ----------------------------------------------------------------- OaA bwd_filter
def oaa_conv_bwd_filter(x, dy, n, crop="valid", P=None, use_numpy_fft=False, b=None):
    """dw[k,c,u,v] = Σ_b Σ_a x[b,c,a] G[b,k,a+(u,v)] ("the change in weight",
    PAPER.md:89) by overlap-and-add in the frequency domain:

      for every n×n block s of dy (origin q_s) take the (2n−1)² window ξ_s of x that
      starts at q_s + o − (n−1) (zero outside x); then
          dŴ[k,c] = Σ_{b,s} conj(DFT_P(dy block)) ⊙ DFT_P(ξ_s)
          r = IDFT_P(dŴ);  dw[k,c,u,v] = r[k,c,n−1−u,n−1−v]
    which is exact for P ≥ 2n−1 (no circular wrap of the lags used).
    n may be an int or a (rows, cols) pair.  b: dy block size (default n; with b×b blocks the
    windows are (b+n−1)² at the same origins q_s + o − (n−1), exact for P ≥ b+n−1 -- reading R18).
    """
    x = np.asarray(x, dtype=np.float64)
    dy = np.asarray(dy, dtype=np.float64)
    nr, nc = (n, n) if np.isscalar(n) else n
    B, C, Nr, Nc = x.shape
    K = dy.shape[1]
    orr, oc = crop_offset(nr, crop), crop_offset(nc, crop)
    br, bc = (nr, nc) if b is None else ((b, b) if np.isscalar(b) else b)
    P1, P2 = _grid(nr, nc, P, b)
    blocks, origins = partition_blocks(dy, br, bc)                    # [B,K,T1,T2,br,bc]
    T1, T2 = blocks.shape[2], blocks.shape[3]
    Gh = dy_spec = dft2(blocks, P1, P2, use_numpy_fft)                # [B,K,T1,T2,P1,P2]
    # x windows: xi_s[i] = x[q_s + o − (n−1) + i], i ∈ [0, b+n−1)²
    Wr, Wc = br + nr - 1, bc + nc - 1
    xpad = np.zeros((B, C, Nr + 2 * T1 * br + 2 * Wr, Nc + 2 * T2 * bc + 2 * Wc))
    shr, shc = Wr, Wc                                                 # shift so indices are >= 0
    xpad[:, :, shr:shr + Nr, shc:shc + Nc] = x
    win = np.zeros((B, C, T1, T2, Wr, Wc))
    for t1 in range(T1):
        for t2 in range(T2):
            r0 = t1 * br + orr - (nr - 1) + shr
            c0 = t2 * bc + oc - (nc - 1) + shc
            win[:, :, t1, t2] = xpad[:, :, r0:r0 + Wr, c0:c0 + Wc]
    Xh = dft2(win, P1, P2, use_numpy_fft)                             # [B,C,T1,T2,P1,P2]
    dWh = np.einsum("bkstfg,bcstfg->kcfg", np.conj(Gh), Xh)           # Σ over b and blocks
    r = idft2(dWh, use_numpy_fft).real                                # [K,C,P1,P2]
    dw = r[:, :, nr - 1::-1, nc - 1::-1][:, :, :nr, :nc]              # lag (n−1−u, n−1−v)
    del dy_spec
    return np.ascontiguousarray(dw)


# ---------------------------------------------------------------- overlap-and-save
def oas_conv_fwd(x, w, crop="valid", P=None, use_numpy_fft=False, keep_aliased=False):
    """y = crop(x * w) by OVERLAP-AND-SAVE, the variant PAPER.md:15 (§1) names beside OaA
    ("the overlap-and-save ... is a similar technique that may be marginally faster but
    has the same complexity"; the paper gives no further detail, so this follows the
    textbook method it cites, Oppenheim & Schafer: overlapping input segments, circular
    convolution by DFT, the aliased samples discarded):

      1. partition the cropped output into ceil(M/n)² n×n blocks (edge blocks clipped);
      2. output block t (rows/cols t·n .. t·n+n−1 of the crop, i.e. t·n + o of the Full
         frame) needs the input segment of (2n−1)² samples starting at t·n + o − (n−1)
         (zero outside x): the segments of neighbouring blocks overlap by n−1;
      3. P-point circular convolution (P ≥ 2n−1, default 2n−1) of every segment with the
         kernel: IDFT_P(DFT_P(segment) ⊙ DFT_P(kernel)), summed over the C channels;
      4. discard the first n−1 samples per axis (wrapped around: aliased) and keep samples
         n−1 .. 2n−2, which equal the linear convolution; write them to the block.
    keep_aliased=True instead returns, per block, the circular result's FIRST n samples
    (the discarded, aliased ones) -- used by the tests to show step 4 is necessary.
    x[B,C,R,Cc], w[K,C,nr,nc]; square blocks per axis as for OaA."""
    x = np.asarray(x, dtype=np.float64)
    w = np.asarray(w, dtype=np.float64)
    B, C, R, Cc = x.shape
    K, C2, nr, nc = w.shape
    assert C == C2
    Mr, Mc = out_size(R, nr, crop), out_size(Cc, nc, crop)
    orr, oc = crop_offset(nr, crop), crop_offset(nc, crop)
    Sr, Sc = 2 * nr - 1, 2 * nc - 1                                   # segment sides
    P1 = Sr if P is None else (P if np.isscalar(P) else P[0])
    P2 = Sc if P is None else (P if np.isscalar(P) else P[1])
    T1, T2 = math.ceil(Mr / nr), math.ceil(Mc / nc)                   # step 1
    pad_r, pad_c = Sr + T1 * nr, Sc + T2 * nc
    xpad = np.zeros((B, C, R + 2 * pad_r, Cc + 2 * pad_c))
    xpad[:, :, pad_r:pad_r + R, pad_c:pad_c + Cc] = x
    seg = np.zeros((B, C, T1, T2, Sr, Sc))
    for t1 in range(T1):                                              # step 2
        for t2 in range(T2):
            r0 = t1 * nr + orr - (nr - 1) + pad_r
            c0 = t2 * nc + oc - (nc - 1) + pad_c
            seg[:, :, t1, t2] = xpad[:, :, r0:r0 + Sr, c0:c0 + Sc]
    Sh = dft2(seg, P1, P2, use_numpy_fft)                             # step 3
    Wh = dft2(w, P1, P2, use_numpy_fft)
    circ = idft2(np.einsum("kcfg,bcstfg->bkstfg", Wh, Sh), use_numpy_fft).real
    y = np.zeros((B, K, T1 * nr, T2 * nc))
    for t1 in range(T1):                                              # step 4
        for t2 in range(T2):
            if keep_aliased:
                blk = circ[:, :, t1, t2, 0:nr, 0:nc]
            else:
                blk = circ[:, :, t1, t2, nr - 1:nr - 1 + nr, nc - 1:nc - 1 + nc]
            y[:, :, t1 * nr:(t1 + 1) * nr, t2 * nc:(t2 + 1) * nc] = blk
    return y[:, :, :Mr, :Mc]


# --------------------------------------------------------------------- FFTconv
def fft_conv_fwd(x, w, crop="valid"):
    """FFTconv: pad input and kernel to next_pow2(N+n−1) per side, FFT, Hadamard,
    inverse, real part, crop.  Uses numpy's FFT
    (a library primitive) at the radix-2 size SPEC.md:265 prescribes."""
    x = np.asarray(x, dtype=np.float64)
    w = np.asarray(w, dtype=np.float64)
    B, C, R, Cc = x.shape
    K, _, nr, nc = w.shape
    P1, P2 = next_pow2(R + nr - 1), next_pow2(Cc + nc - 1)
    Xh = dft2(x, P1, P2, use_numpy_fft=True)
    Wh = dft2(w, P1, P2, use_numpy_fft=True)
    Yh = np.einsum("kcfg,bcfg->bkfg", Wh, Xh)
    full = idft2(Yh, use_numpy_fft=True).real[:, :, :R + nr - 1, :Cc + nc - 1]
    return _crop(full, R, Cc, nr, nc, crop)


def oaa_block_count(N: int, n: int) -> int:
    """ceil(N/n)² blocks per channel (reading R1)."""
    return math.ceil(N / n) ** 2
