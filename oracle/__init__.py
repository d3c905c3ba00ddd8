"""CPU float64 oracle for the OaA convolution layer (arXiv 1601.06815).

TEST INFRASTRUCTURE -- not product code.  Only tests/, ``__graft_entry__.smoke()`` and
bench.py's ``cpu_baseline`` / ``--impl reference`` leg may import this package.  The
product path (paper_1601_06815_b200) never imports it and shares no code with it.

Contents
  * liboracle.so (oracle/oracle.c): the plain DIRECT definitions of forward, bwd_data
    and bwd_filter in fp64 with OpenMP over independent outputs, plus sampled
    single-element evaluation on fp32 inputs for full-size parity checks.
  * oaa_ref.py: the paper's overlap-and-add algorithm step by step (fp64, plain DFT
    matrices or numpy FFT), FFTconv, block partition.

Pins (what ties this oracle to something other than itself) live in
tests/test_oracle_*.py; see DESIGN.md §"Oracle" for the list.  Functions with no pin:
none ("parity unpinned" would be stated here).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

from . import oaa_ref  # noqa: F401  (re-export)

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

CROP = {"full": 0, "valid": 1, "same": 2}


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc -O2 -fopenmp (building the checker is not using it)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-fopenmp", "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm"]
        subprocess.run(cmd, check=True)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            dp = ctypes.POINTER(ctypes.c_double)
            fp = ctypes.POINTER(ctypes.c_float)
            i64p = ctypes.POINTER(ctypes.c_int64)
            I = ctypes.c_int
            for name in ("oracle_conv_fwd", "oracle_conv_bwd_data", "oracle_conv_bwd_filter"):
                f = getattr(L, name)
                f.argtypes = [dp, dp, dp, I, I, I, I, I, I, I]
                f.restype = I
            for name in ("oracle_conv_fwd_rect", "oracle_conv_bwd_data_rect",
                         "oracle_conv_bwd_filter_rect"):
                f = getattr(L, name)
                f.argtypes = [dp, dp, dp, I, I, I, I, I, I, I, I, I]
                f.restype = I
            for name in ("oracle_fwd_sample", "oracle_bwd_data_sample", "oracle_bwd_filter_sample"):
                f = getattr(L, name)
                f.argtypes = [fp, fp, I, I, I, I, I, I, i64p, ctypes.c_long, dp, I]
                f.restype = I
            L.oracle_step_f32.argtypes = [fp, fp, fp, dp, dp, dp, I, I, I, I, I, I, I]
            L.oracle_step_f32.restype = I
            L.oracle_out_size.argtypes = [I, I, I]
            L.oracle_out_size.restype = I
            L.oracle_crop_offset.argtypes = [I, I]
            L.oracle_crop_offset.restype = I
            L.oracle_max_threads.argtypes = []
            L.oracle_max_threads.restype = I
            _lib = L
    return _lib


def _crop_id(crop) -> int:
    return CROP[crop] if isinstance(crop, str) else int(crop)


def _dptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _fptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))


def out_size(N: int, n: int, crop) -> int:
    return lib().oracle_out_size(int(N), int(n), _crop_id(crop))


def max_threads() -> int:
    return lib().oracle_max_threads()


def _rect(a):
    return a.shape[-2], a.shape[-1]


def conv_fwd(x, w, crop="valid", nthreads: int = 0) -> np.ndarray:
    """Direct fp64 forward.  x[B,C,R,Cc], w[K,C,nr,nc] (any float dtype, promoted)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    w = np.ascontiguousarray(w, dtype=np.float64)
    B, C, R, Cc = x.shape
    K, C2, nr, nc = w.shape
    assert C == C2
    cid = _crop_id(crop)
    Mr, Mc = lib().oracle_out_size(R, nr, cid), lib().oracle_out_size(Cc, nc, cid)
    if Mr < 1 or Mc < 1:
        raise ValueError("invalid crop for these shapes")
    y = np.zeros((B, K, Mr, Mc))
    rc = lib().oracle_conv_fwd_rect(_dptr(x), _dptr(w), _dptr(y), B, C, K, R, Cc, nr, nc, cid, nthreads)
    assert rc == 0
    return y


def conv_bwd_data(dy, w, N, crop="valid", nthreads: int = 0) -> np.ndarray:
    """Direct fp64 data gradient dx[B,C,N,N] (N may be (rows, cols))."""
    dy = np.ascontiguousarray(dy, dtype=np.float64)
    w = np.ascontiguousarray(w, dtype=np.float64)
    B, K, _, _ = dy.shape
    K2, C, nr, nc = w.shape
    assert K == K2
    R, Cc = (N, N) if np.isscalar(N) else N
    cid = _crop_id(crop)
    assert dy.shape[2:] == (lib().oracle_out_size(R, nr, cid), lib().oracle_out_size(Cc, nc, cid))
    dx = np.zeros((B, C, R, Cc))
    rc = lib().oracle_conv_bwd_data_rect(_dptr(dy), _dptr(w), _dptr(dx), B, C, K, R, Cc, nr, nc, cid, nthreads)
    assert rc == 0
    return dx


def conv_bwd_filter(x, dy, n, crop="valid", nthreads: int = 0) -> np.ndarray:
    """Direct fp64 weight gradient dw[K,C,n,n] summed over the batch (n may be a pair)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    dy = np.ascontiguousarray(dy, dtype=np.float64)
    B, C, R, Cc = x.shape
    B2, K, _, _ = dy.shape
    assert B == B2
    nr, nc = (n, n) if np.isscalar(n) else n
    cid = _crop_id(crop)
    assert dy.shape[2:] == (lib().oracle_out_size(R, nr, cid), lib().oracle_out_size(Cc, nc, cid))
    dw = np.zeros((K, C, nr, nc))
    rc = lib().oracle_conv_bwd_filter_rect(_dptr(x), _dptr(dy), _dptr(dw), B, C, K, R, Cc, nr, nc, cid, nthreads)
    assert rc == 0
    return dw


def _sample(fn, a, b, dims, crop, idx, nthreads):
    a = np.ascontiguousarray(a, dtype=np.float32)
    b = np.ascontiguousarray(b, dtype=np.float32)
    idx = np.ascontiguousarray(idx, dtype=np.int64).reshape(-1, 4)
    out = np.zeros(idx.shape[0])
    rc = fn(_fptr(a), _fptr(b), *dims, _crop_id(crop),
            idx.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), idx.shape[0], _dptr(out), nthreads)
    if rc != 0:
        raise ValueError(f"oracle sample failed rc={rc}")
    return out


def fwd_sample(x, w, crop, idx, nthreads: int = 0):
    """y at (b,k,i,j) tuples, evaluated one by one from the fp32 inputs."""
    B, C, N, _ = x.shape
    K, _, n, _ = w.shape
    return _sample(lib().oracle_fwd_sample, x, w, (B, C, K, N, n), crop, idx, nthreads)


def bwd_data_sample(dy, w, N, crop, idx, nthreads: int = 0):
    """dx at (b,c,a1,a2) tuples."""
    B, K, _, _ = dy.shape
    _, C, n, _ = w.shape
    return _sample(lib().oracle_bwd_data_sample, dy, w, (B, C, K, N, n), crop, idx, nthreads)


def bwd_filter_sample(x, dy, n, crop, idx, nthreads: int = 0):
    """dw at (k,c,u,v) tuples (each a sum over the whole batch)."""
    B, C, N, _ = x.shape
    K = dy.shape[1]
    return _sample(lib().oracle_bwd_filter_sample, x, dy, (B, C, K, N, n), crop, idx, nthreads)


def step_f32(x, w, dy, crop="valid", nthreads: int = 0):
    """One fwd + bwd_data + bwd_filter of the direct definitions on fp32 inputs."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    w = np.ascontiguousarray(w, dtype=np.float32)
    dy = np.ascontiguousarray(dy, dtype=np.float32)
    B, C, N, _ = x.shape
    K, _, n, _ = w.shape
    M = dy.shape[-1]
    y = np.zeros((B, K, M, M))
    dx = np.zeros((B, C, N, N))
    dw = np.zeros((K, C, n, n))
    rc = lib().oracle_step_f32(_fptr(x), _fptr(w), _fptr(dy), _dptr(y), _dptr(dx), _dptr(dw),
                               B, C, K, N, n, _crop_id(crop), nthreads)
    assert rc == 0
    return y, dx, dw
