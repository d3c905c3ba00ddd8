"""B200-native overlap-and-add (OaA) convolution layer (arXiv 1601.06815).

Thin Python binding over the C ABI of ``liboaa.so`` (include/oaa.h).  Every step of the
layer -- tiling, zero-padding, block FFTs, per-bin channel contraction, inverse FFT,
overlap-add, crop -- runs in the library's sm_100a kernels; this module only checks
tensors, allocates outputs / workspaces through PyTorch's caching allocator and passes
raw device pointers plus the current CUDA stream.  There is no CPU fallback: if the
extension is missing or a tensor is not on a CUDA device the call raises.

    import paper_1601_06815_b200 as oaa
    y  = oaa.conv_fwd(x, w, crop="valid")            # x[B,C,N,N], w[K,C,n,n] -> y[B,K,M,M]
    dx = oaa.conv_bwd_data(dy, w, N, crop="valid")   # -> dx[B,C,N,N]
    dw = oaa.conv_bwd_filter(x, dy, n, crop="valid") # -> dw[K,C,n,n] (sum over the batch)
    layer = oaa.OaAConv2d(C, K, n)                    # autograd module (true convolution)
"""
from __future__ import annotations

import ctypes
import os
import threading
from typing import Optional

import torch

__all__ = [
    "conv_fwd", "conv_bwd_data", "conv_bwd_filter", "out_size", "workspace_bytes", "lib",
    "OaAConv2dFunction", "OaAConv2d", "launch_count", "profile_enable", "profile_collect",
    "profile_collect_kernels",
    "CROPS", "block_size", "OP_FWD", "OP_BWD_DATA", "OP_BWD_FILTER", "OP_FWD_OAS", "OP_BWD", "OaAError", "conv_fwd_oas", "PreparedWeights", "conv_bwd",
]

_PKG = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.environ.get("OAA_LIB") or os.path.join(_PKG, "liboaa.so")  # OAA_LIB: experiment builds
CROPS = {"full": 0, "valid": 1, "same": 2}
OP_FWD, OP_BWD_DATA, OP_BWD_FILTER, OP_FWD_OAS, OP_BWD = 0, 1, 2, 3, 4
_STATUS = {0: "OAA_OK", 1: "OAA_ERR_INVALID_VALUE", 2: "OAA_ERR_UNSUPPORTED",
           3: "OAA_ERR_WORKSPACE", 4: "OAA_ERR_CUDA"}

_lock = threading.Lock()
_lib = None


class OaAError(RuntimeError):
    pass


def lib():
    """The loaded liboaa.so (ctypes).  Raises if the extension has not been built."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(_LIB_PATH):
                raise OaAError(f"{_LIB_PATH} missing: run `python -m paper_1601_06815_b200.build` "
                               "(there is no CPU fallback)")
            L = ctypes.CDLL(_LIB_PATH)
            I, Z, V, F = ctypes.c_int, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p
            L.oaa_conv_out_size.argtypes = [I, I, I]
            L.oaa_conv_out_size.restype = I
            L.oaa_conv_workspace_bytes.argtypes = [I, I, I, I, I, I, I]
            L.oaa_conv_workspace_bytes.restype = Z
            for name in ("oaa_conv_fwd", "oaa_conv_bwd_data", "oaa_conv_bwd_filter", "oaa_conv_fwd_oas"):
                f = getattr(L, name)
                f.argtypes = [F, F, F, I, I, I, I, I, I, V, Z, V]
                f.restype = I
            L.oaa_conv_bwd.argtypes = [F, F, F, F, F, I, I, I, I, I, I, V, Z, V]
            L.oaa_conv_bwd.restype = I
            L.oaa_weight_spectra_bytes.argtypes = [I, I, I, I, I, I]
            L.oaa_weight_spectra_bytes.restype = Z
            L.oaa_weight_spectra.argtypes = [I, F, V, Z, I, I, I, I, I, V]
            L.oaa_weight_spectra.restype = I
            for name in ("oaa_conv_fwd_prepared", "oaa_conv_bwd_data_prepared"):
                f = getattr(L, name)
                f.argtypes = [F, V, F, I, I, I, I, I, I, V, Z, V]
                f.restype = I
            L.oaa_debug_bin_gemm_workspace_bytes.argtypes = [I, I, I, I]
            L.oaa_debug_bin_gemm_workspace_bytes.restype = Z
            L.oaa_debug_bin_gemm.argtypes = [F, F, F, I, I, I, I, V, Z, V]
            L.oaa_debug_bin_gemm.restype = I
            L.oaa_status_string.argtypes = [I]
            L.oaa_status_string.restype = ctypes.c_char_p
            L.oaa_block_size.argtypes = [I, I, I, I, I, I]
            L.oaa_block_size.restype = I
            L.oaa_version.argtypes = []
            L.oaa_version.restype = ctypes.c_char_p
            L.oaa_launch_count.argtypes = []
            L.oaa_launch_count.restype = ctypes.c_uint64
            L.oaa_profile_enable.argtypes = [I]
            L.oaa_profile_enable.restype = None
            L.oaa_profile_collect.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int)]
            L.oaa_profile_collect.restype = I
            L.oaa_profile_kernel_count.argtypes = []
            L.oaa_profile_kernel_count.restype = I
            L.oaa_profile_kernel_name.argtypes = [I]
            L.oaa_profile_kernel_name.restype = ctypes.c_char_p
            L.oaa_profile_collect_kernels.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int), I]
            L.oaa_profile_collect_kernels.restype = I
            _lib = L
    return _lib


def version() -> str:
    return lib().oaa_version().decode()


def block_size(op: str, C: int, K: int, N: int, n: int, crop: str = "valid") -> int:
    """Block size b the fwd / bwd_data call tiles into (host planning only; R18)."""
    if op not in ("fwd", "bwd_data"):
        raise ValueError("op must be 'fwd' or 'bwd_data'")
    return lib().oaa_block_size(OP_FWD if op == "fwd" else OP_BWD_DATA, int(C), int(K), int(N), int(n), _crop_id(crop))


def _crop_id(crop) -> int:
    if isinstance(crop, str):
        if crop not in CROPS:
            raise ValueError(f"crop must be one of {list(CROPS)}")
        return CROPS[crop]
    return int(crop)


def out_size(N: int, n: int, crop="valid") -> int:
    M = lib().oaa_conv_out_size(int(N), int(n), _crop_id(crop))
    if M < 1:
        raise ValueError(f"invalid (N={N}, n={n}, crop={crop})")
    return M


def workspace_bytes(op: int, B: int, C: int, K: int, N: int, n: int, crop="valid") -> int:
    return int(lib().oaa_conv_workspace_bytes(int(op), B, C, K, N, n, _crop_id(crop)))


# --------------------------------------------------------------------- workspaces
_ws_cache: dict = {}


def _workspace(nbytes: int, device: torch.device, stream: torch.cuda.Stream) -> torch.Tensor:
    """Per-(device, stream) cached workspace, allocated ON `stream` so the caching
    allocator orders its reuse after the kernels that stream runs on it."""
    key = (device.index, stream.cuda_stream)
    ws = _ws_cache.get(key)
    if ws is None or ws.numel() < nbytes:
        _ws_cache.pop(key, None)  # freed on `stream`: reused only after its kernels
        with torch.cuda.stream(stream):
            ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
        _ws_cache[key] = ws
    return ws


def _check(t: torch.Tensor, name: str, ndim: int = 4) -> None:
    if not isinstance(t, torch.Tensor):
        raise ValueError(f"{name} must be a torch.Tensor")
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU path)")
    if t.dtype != torch.float32:
        raise ValueError(f"{name} must be float32, got {t.dtype}")
    if t.dim() != ndim:
        raise ValueError(f"{name} must be {ndim}-D, got shape {tuple(t.shape)}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


def _call(fn, a, b, out, dims, crop, op, stream):
    B, C, K, N, n = dims
    dev = out.device
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    nbytes = workspace_bytes(op, B, C, K, N, n, crop)
    ws = _workspace(nbytes, dev, s)
    if s != torch.cuda.current_stream(dev):
        # the kernels run on `s`, the tensors were allocated on the current stream: tell
        # the caching allocator, so a block freed early is not handed out while `s` still
        # reads or writes it
        for t in (a, b, out):
            t.record_stream(s)
    st = fn(ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(b.data_ptr()),
            ctypes.c_void_p(out.data_ptr()), B, C, K, N, n, _crop_id(crop),
            ctypes.c_void_p(ws.data_ptr()), ctypes.c_size_t(ws.numel()), ctypes.c_void_p(s.cuda_stream))
    if st != 0:
        msg = lib().oaa_status_string(st).decode()
        if st in (1, 2, 3):
            raise ValueError(msg)
        raise OaAError(msg)
    return out


def conv_fwd(x: torch.Tensor, w: torch.Tensor, crop="valid", out: Optional[torch.Tensor] = None,
             stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """y[B,K,M,M] = crop(Σ_c x[:,c] ∗ w[:,c]) (true convolution)."""
    _check(x, "x"); _check(w, "w")
    B, C, N, N2 = x.shape
    K, C2, n, n2 = w.shape
    if N != N2 or n != n2:
        raise ValueError("square images and kernels only")
    if C != C2:
        raise ValueError(f"channel mismatch: x has C={C}, w has C={C2}")
    if x.device != w.device:
        raise ValueError("x and w on different devices")
    M = out_size(N, n, crop)
    if out is None:
        out = torch.empty((B, K, M, M), dtype=torch.float32, device=x.device)
    else:
        _check(out, "out")
        if tuple(out.shape) != (B, K, M, M):
            raise ValueError(f"out must have shape {(B, K, M, M)}")
    return _call(lib().oaa_conv_fwd, x, w, out, (B, C, K, N, n), crop, OP_FWD, stream)


def conv_fwd_oas(x: torch.Tensor, w: torch.Tensor, crop="valid", out: Optional[torch.Tensor] = None,
                 stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """The same y as conv_fwd, by overlap-and-save (include/oaa.h): each
    n×n output block is the alias-free part of a (2n−1)-point circular convolution of its
    input window.  C ≤ 4 (SIMT walker) or C, K ≥ 16 (tensor-core path)."""
    _check(x, "x"); _check(w, "w")
    B, C, N, N2 = x.shape
    K, C2, n, n2 = w.shape
    if N != N2 or n != n2:
        raise ValueError("square images and kernels only")
    if C != C2:
        raise ValueError(f"channel mismatch: x has C={C}, w has C={C2}")
    M = out_size(N, n, crop)
    if out is None:
        out = torch.empty((B, K, M, M), dtype=torch.float32, device=x.device)
    else:
        _check(out, "out")
        if tuple(out.shape) != (B, K, M, M):
            raise ValueError(f"out must have shape {(B, K, M, M)}")
    return _call(lib().oaa_conv_fwd_oas, x, w, out, (B, C, K, N, n), crop, OP_FWD_OAS, stream)


def conv_bwd_data(dy: torch.Tensor, w: torch.Tensor, N: int, crop="valid",
                  out: Optional[torch.Tensor] = None,
                  stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """dx[B,C,N,N]: the error propagated through the layer."""
    _check(dy, "dy"); _check(w, "w")
    B, K, M, M2 = dy.shape
    K2, C, n, n2 = w.shape
    if K != K2:
        raise ValueError(f"channel mismatch: dy has K={K}, w has K={K2}")
    if M != M2 or n != n2:
        raise ValueError("square maps and kernels only")
    if M != out_size(N, n, crop):
        raise ValueError(f"dy side {M} != out_size(N={N}, n={n}, {crop})")
    if out is None:
        out = torch.empty((B, C, N, N), dtype=torch.float32, device=dy.device)
    else:
        _check(out, "out")
        if tuple(out.shape) != (B, C, N, N):
            raise ValueError(f"out must have shape {(B, C, N, N)}")
    return _call(lib().oaa_conv_bwd_data, dy, w, out, (B, C, K, N, n), crop, OP_BWD_DATA, stream)


def conv_bwd_filter(x: torch.Tensor, dy: torch.Tensor, n: int, crop="valid",
                    out: Optional[torch.Tensor] = None,
                    stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """dw[K,C,n,n] = Σ over the batch: the change in weight."""
    _check(x, "x"); _check(dy, "dy")
    B, C, N, N2 = x.shape
    B2, K, M, M2 = dy.shape
    if B != B2:
        raise ValueError("batch mismatch")
    if N != N2 or M != M2:
        raise ValueError("square maps only")
    if M != out_size(N, n, crop):
        raise ValueError(f"dy side {M} != out_size(N={N}, n={n}, {crop})")
    if out is None:
        out = torch.empty((K, C, n, n), dtype=torch.float32, device=x.device)
    else:
        _check(out, "out")
        if tuple(out.shape) != (K, C, n, n):
            raise ValueError(f"out must have shape {(K, C, n, n)}")
    return _call(lib().oaa_conv_bwd_filter, x, dy, out, (B, C, K, N, n), crop, OP_BWD_FILTER, stream)


def conv_bwd(x: torch.Tensor, dy: torch.Tensor, w: torch.Tensor, crop="valid",
             dx: Optional[torch.Tensor] = None, dw: Optional[torch.Tensor] = None,
             stream: Optional[torch.cuda.Stream] = None):
    """(dx, dw) in one call -- the two backward convolutions of PAPER.md:89 (include/oaa.h
    oaa_conv_bwd; on the tensor-core path the dy spectra are computed once for both)."""
    _check(x, "x"); _check(dy, "dy"); _check(w, "w")
    B, C, N, N2 = x.shape
    B2, K, M, M2 = dy.shape
    K2, C2, n, n2 = w.shape
    if B != B2 or K != K2 or C != C2 or N != N2 or M != M2 or n != n2:
        raise ValueError("shape mismatch")
    if M != out_size(N, n, crop):
        raise ValueError(f"dy side {M} != out_size(N={N}, n={n}, {crop})")
    dx = torch.empty_like(x) if dx is None else dx
    dw = torch.empty_like(w) if dw is None else dw
    _check(dx, "dx"); _check(dw, "dw")
    if dx.shape != x.shape or dw.shape != w.shape:
        raise ValueError("dx / dw shapes")
    dev = x.device
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    ws = _workspace(workspace_bytes(OP_BWD, B, C, K, N, n, crop), dev, s)
    if s != torch.cuda.current_stream(dev):
        for t in (x, dy, w, dx, dw):
            t.record_stream(s)
    P = ctypes.c_void_p
    st = lib().oaa_conv_bwd(P(x.data_ptr()), P(dy.data_ptr()), P(w.data_ptr()), P(dx.data_ptr()), P(dw.data_ptr()),
                            B, C, K, N, n, _crop_id(crop), P(ws.data_ptr()), ctypes.c_size_t(ws.numel()),
                            P(s.cuda_stream))
    if st != 0:
        msg = lib().oaa_status_string(st).decode()
        raise (ValueError if st in (1, 2, 3) else OaAError)(msg)
    return dx, dw


def debug_bin_gemm(A: torch.Tensor, B: torch.Tensor) -> torch.Tensor:
    """D[f] = A[f] @ B[f].T with the tcgen05 3×TF32 contraction kernel (diagnostics)."""
    _check(A, "A", 3); _check(B, "B", 3)
    F, M, Kd = A.shape
    F2, N, Kd2 = B.shape
    if F != F2 or Kd != Kd2:
        raise ValueError("shape mismatch")
    D = torch.empty((F, M, N), dtype=torch.float32, device=A.device)
    s = torch.cuda.current_stream(A.device)
    nbytes = int(lib().oaa_debug_bin_gemm_workspace_bytes(F, M, N, Kd))
    ws = torch.empty(nbytes, dtype=torch.uint8, device=A.device)
    st = lib().oaa_debug_bin_gemm(ctypes.c_void_p(A.data_ptr()), ctypes.c_void_p(B.data_ptr()),
                                  ctypes.c_void_p(D.data_ptr()), F, M, N, Kd, ctypes.c_void_p(ws.data_ptr()),
                                  nbytes, ctypes.c_void_p(s.cuda_stream))
    if st != 0:
        raise OaAError(lib().oaa_status_string(st).decode())
    return D


def launch_count() -> int:
    """Kernels launched through liboaa.so by this process so far."""
    return int(lib().oaa_launch_count())


def profile_enable(on: bool = True) -> None:
    lib().oaa_profile_enable(1 if on else 0)


def profile_collect():
    """Summed main-kernel milliseconds and launch counts per op since the last collect:
    ({'fwd': ms, 'bwd_data': ms, 'bwd_filter': ms}, {...counts})."""
    ms = (ctypes.c_double * 3)()
    cnt = (ctypes.c_int * 3)()
    r = lib().oaa_profile_collect(ms, cnt)
    if r < 0:
        raise OaAError("oaa_profile_collect: CUDA error")
    names = ("fwd", "bwd_data", "bwd_filter")
    return {k: ms[i] for i, k in enumerate(names)}, {k: cnt[i] for i, k in enumerate(names)}


def profile_collect_kernels():
    """Summed milliseconds and launch counts per kernel since the last collect:
    ({'walk': ms, ...}, {'walk': count, ...}), only kernels that ran."""
    L = lib()
    n = L.oaa_profile_kernel_count()
    ms = (ctypes.c_double * n)()
    cnt = (ctypes.c_int * n)()
    if L.oaa_profile_collect_kernels(ms, cnt, n) < 0:
        raise OaAError("oaa_profile_collect_kernels: CUDA error")
    names = [L.oaa_profile_kernel_name(i).decode() for i in range(n)]
    return ({names[i]: ms[i] for i in range(n) if cnt[i]}, {names[i]: cnt[i] for i in range(n) if cnt[i]})


# ------------------------------------------------------------ prepared weight spectra
class PreparedWeights:
    """Weight spectra computed once and reused across calls (include/oaa.h, NEXT-4 of
    SURVEY.md §8(f)): ``pw = PreparedWeights(w, N, op="fwd")`` then ``pw.fwd(x)`` (or
    ``pw.bwd_data(dy)`` for op="bwd_data").  Results are bitwise those of conv_fwd /
    conv_bwd_data with the same w.  Re-create after changing w."""

    def __init__(self, w: torch.Tensor, N: int, op: str = "fwd", crop="valid",
                 stream: Optional[torch.cuda.Stream] = None):
        _check(w, "w")
        if op not in ("fwd", "bwd_data"):
            raise ValueError("op must be 'fwd' or 'bwd_data'")
        self.op, self.crop, self.N = op, crop, int(N)
        self.K, self.C, self.n = w.shape[0], w.shape[1], w.shape[2]
        opc = OP_FWD if op == "fwd" else OP_BWD_DATA
        nbytes = int(lib().oaa_weight_spectra_bytes(opc, self.C, self.K, self.N, self.n, _crop_id(crop)))
        if nbytes == 0:
            raise ValueError("unsupported arguments")
        s = stream if stream is not None else torch.cuda.current_stream(w.device)
        with torch.cuda.stream(s):
            self.spec = torch.empty(nbytes, dtype=torch.uint8, device=w.device)
        st = lib().oaa_weight_spectra(opc, ctypes.c_void_p(w.data_ptr()), ctypes.c_void_p(self.spec.data_ptr()),
                                      ctypes.c_size_t(nbytes), self.C, self.K, self.N, self.n, _crop_id(crop),
                                      ctypes.c_void_p(s.cuda_stream))
        if st != 0:
            raise OaAError(lib().oaa_status_string(st).decode())

    def fwd(self, x: torch.Tensor, out: Optional[torch.Tensor] = None,
            stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
        if self.op != "fwd":
            raise ValueError("prepared for bwd_data")
        _check(x, "x")
        B, C, N, _ = x.shape
        if C != self.C or N != self.N:
            raise ValueError("x does not match the prepared (C, N)")
        M = out_size(N, self.n, self.crop)
        out = out if out is not None else torch.empty((B, self.K, M, M), device=x.device)
        return _call(lib().oaa_conv_fwd_prepared, x, self.spec, out, (B, self.C, self.K, N, self.n),
                     self.crop, OP_FWD, stream)

    def bwd_data(self, dy: torch.Tensor, out: Optional[torch.Tensor] = None,
                 stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
        if self.op != "bwd_data":
            raise ValueError("prepared for fwd")
        _check(dy, "dy")
        B, K, M, _ = dy.shape
        if K != self.K or M != out_size(self.N, self.n, self.crop):
            raise ValueError("dy does not match the prepared (K, N)")
        out = out if out is not None else torch.empty((B, self.C, self.N, self.N), device=dy.device)
        return _call(lib().oaa_conv_bwd_data_prepared, dy, self.spec, out, (B, self.C, self.K, self.N, self.n),
                     self.crop, OP_BWD_DATA, stream)


# --------------------------------------------------------------------- autograd
class OaAConv2dFunction(torch.autograd.Function):
    """y = OaA conv(x, w); backward = the two OaA convolutions of PAPER.md:89."""

    @staticmethod
    def forward(ctx, x, w, crop="valid"):
        x = x.contiguous(); w = w.contiguous()
        ctx.save_for_backward(x, w)
        ctx.crop = crop
        return conv_fwd(x, w, crop)

    @staticmethod
    def backward(ctx, dy):
        x, w = ctx.saved_tensors
        dy = dy.contiguous()
        dx = dw = None
        if ctx.needs_input_grad[0]:
            dx = conv_bwd_data(dy, w, x.shape[-1], ctx.crop)
        if ctx.needs_input_grad[1]:
            dw = conv_bwd_filter(x, dy, w.shape[-1], ctx.crop)
        return dx, dw, None


class OaAConv2d(torch.nn.Module):
    """Convolutional layer with K kernels of C×n×n, stride 1, no bias
    (reading R12), true convolution, output crop Full/Valid/Same."""

    def __init__(self, C: int, K: int, n: int, crop: str = "valid", device=None):
        super().__init__()
        self.crop = crop
        w = torch.empty(K, C, n, n, device=device, dtype=torch.float32)
        torch.nn.init.kaiming_uniform_(w, a=5 ** 0.5)
        self.weight = torch.nn.Parameter(w)

    def forward(self, x):
        return OaAConv2dFunction.apply(x, self.weight, self.crop)
