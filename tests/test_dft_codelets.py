"""The product's register DFT codelets (csrc/dft.cuh), built for the host, against
numpy's FFT (a library routine): every odd P = 2n−1 ≤ 15, both signs, the pruned
(n leading non-zero inputs) forward variant, and the Hermitian half → real inverse."""
import ctypes
import os
import subprocess

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "native", "dft_selftest.cu")
LIB = os.path.join(HERE, "native", "libdft_selftest.so")
DEP = os.path.join(os.path.dirname(HERE), "paper_1601_06815_b200", "csrc", "dft.cuh")


@pytest.fixture(scope="module")
def L():
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(SRC), os.path.getmtime(DEP)):
        subprocess.run(["nvcc", "-std=c++17", "-O2", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC",
                        "-shared", "-o", LIB, SRC], check=True)
    lib = ctypes.CDLL(LIB)
    fp = ctypes.POINTER(ctypes.c_float)
    lib.dft_selftest.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, fp, fp, fp, fp]
    lib.c2r_selftest.argtypes = [ctypes.c_int, fp, fp, fp]
    return lib


def _p(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))


@pytest.mark.parametrize("P", [1, 3, 5, 7, 9, 11, 13, 15])
@pytest.mark.parametrize("sign", [-1, 1])
@pytest.mark.parametrize("pruned", [False, True])
def test_dft_codelet(L, P, sign, pruned):
    rng = np.random.default_rng(P * 10 + sign + 3 * pruned)
    n = (P + 1) // 2
    if pruned and sign > 0:
        pytest.skip("pruned variant is forward only")
    x = (rng.uniform(-1, 1, P) + 1j * rng.uniform(-1, 1, P)).astype(np.complex64)
    if pruned:
        x[n:] = 0
    xr, xi = np.ascontiguousarray(x.real), np.ascontiguousarray(x.imag)
    yr, yi = np.zeros(P, np.float32), np.zeros(P, np.float32)
    assert L.dft_selftest(P, sign, n if pruned else P, _p(xr), _p(xi), _p(yr), _p(yi)) == 0
    ref = np.fft.fft(x.astype(np.complex128)) if sign < 0 else np.fft.ifft(x.astype(np.complex128)) * P
    np.testing.assert_allclose(yr + 1j * yi, ref, atol=5e-6 * P)


@pytest.mark.parametrize("P", [1, 3, 5, 7, 9, 11, 13, 15])
def test_c2r_codelet(L, P):
    rng = np.random.default_rng(P)
    y = rng.uniform(-1, 1, P)
    Z = np.fft.fft(y)  # Hermitian
    H = (P + 1) // 2
    zr = np.ascontiguousarray(Z.real[:H], np.float32)
    zi = np.ascontiguousarray(Z.imag[:H], np.float32)
    out = np.zeros(P, np.float32)
    assert L.c2r_selftest(P, _p(zr), _p(zi), _p(out)) == 0
    np.testing.assert_allclose(out, y * P, atol=5e-6 * P)   # unnormalised inverse
