"""Pins for the step-by-step OaA / FFTconv / DFT references (oracle/oaa_ref.py).

The paper's core correctness claim is that the three methods agree ("create the same
results as a traditional spacial convolution"; Table 2).
We check: OaA == direct == FFTconv (SPEC.md:257 backend equivalence), the block-count
law, n = N convergence, n = 1 degenerating to a
scalar multiply, the P ≥ 2n−1 requirement (aliasing at P = 2n−2,
PAPER.md:85), SPEC's worked examples and the DFT's textbook properties (impulse,
constant, round trip, Parseval, numpy FFT equality).
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
from oracle import oaa_ref

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_worked_examples.json")))
CROPS = ["full", "valid", "same"]
RNG = np.random.default_rng(77)


def rnd(*shape):
    return RNG.uniform(-1, 1, size=shape)


def tol(C, n, ax=1.0, aw=1.0):
    """fp64 tolerance 1e-12·C·n²·max|x|·max|w| (SPEC.md:257 scaled by C)."""
    return 1e-12 * C * n * n * ax * aw


# ------------------------------------------------------------------------------- DFT
@pytest.mark.parametrize("ex", GOLD["dft1d"], ids=lambda e: e["cite"][:11])
def test_dft_spec_examples(ex):
    x = np.array([a + 1j * b for a, b in ex["x"]])
    X = oaa_ref.dft_matrix(len(x), -1) @ x
    np.testing.assert_allclose(X, np.array([a + 1j * b for a, b in ex["X"]]), atol=1e-14)


@pytest.mark.parametrize("P", [1, 2, 3, 5, 7, 8, 9, 13, 15, 16])
def test_dft_properties(P):
    a = rnd(3, P, P) + 1j * rnd(3, P, P)
    A = oaa_ref.dft2(a, P)
    np.testing.assert_allclose(A, np.fft.fft2(a), atol=1e-11)               # library FFT
    np.testing.assert_allclose(oaa_ref.idft2(A), a, atol=1e-12)             # round trip
    np.testing.assert_allclose((np.abs(a) ** 2).sum(), (np.abs(A) ** 2).sum() / (P * P), rtol=1e-12)  # Parseval
    imp = np.zeros((P, P)); imp[0, 0] = 1
    np.testing.assert_allclose(oaa_ref.dft2(imp, P), np.ones((P, P)), atol=1e-14)   # impulse → ones
    np.testing.assert_allclose(oaa_ref.dft2(np.ones((P, P)), P)[0, 0], P * P)       # DC spike
    if P > 1:
        assert np.abs(oaa_ref.dft2(np.ones((P, P)), P).reshape(-1)[1:]).max() < 1e-11


# -------------------------------------------------------------------- partition
@pytest.mark.parametrize("ex", GOLD["partition"], ids=lambda e: e["cite"][:11])
def test_partition_spec_examples(ex):
    a = rnd(ex["N"], ex["N"])
    blocks, origins = oaa_ref.partition_blocks(a, ex["n"])
    assert blocks.shape[0] * blocks.shape[1] == ex["count"] == len(origins)
    assert oaa_ref.oaa_block_count(ex["N"], ex["n"]) == ex["count"]
    if "origins" in ex:
        assert [list(o) for o in origins] == ex["origins"]


@pytest.mark.parametrize("N", range(1, 20))
@pytest.mark.parametrize("n", [1, 2, 3, 5, 8])
def test_partition_reassembles_and_count_law(N, n):
    a = rnd(N, N)
    blocks, origins = oaa_ref.partition_blocks(a, n)
    assert len(origins) == math.ceil(N / n) ** 2
    re = np.zeros((math.ceil(N / n) * n,) * 2)
    for (r, c), blk in zip(origins, blocks.reshape(-1, n, n)):
        re[r:r + n, c:c + n] = blk
    np.testing.assert_array_equal(re[:N, :N], a)
    assert not re[N:, :].any() and not re[:, N:].any()   # zero-filled edge blocks


def test_oaa_spec_block_example():
    ex = GOLD["oaa_blocks"][0]
    x = np.array(ex["x"], float); w = np.array(ex["w"], float)
    blocks, origins = oaa_ref.partition_blocks(x, 1, 2)
    np.testing.assert_array_equal(blocks.reshape(-1, 1, 2), np.array(ex["blocks"], float))
    assert [list(o) for o in origins] == ex["offsets"]
    for blk, bc in zip(blocks.reshape(-1, 1, 2), ex["block_convs"]):
        got = oaa_ref.oaa_conv_fwd(blk[None, None], w[None, None], "full")[0, 0]
        np.testing.assert_allclose(got, np.array(bc, float), atol=1e-13)


@pytest.mark.parametrize("ex", GOLD["conv"], ids=lambda e: e["cite"][:12])
def test_oaa_spec_worked_examples(ex):
    x = np.array(ex["x"], float)[None, None]; w = np.array(ex["w"], float)[None, None]
    np.testing.assert_allclose(oaa_ref.oaa_conv_fwd(x, w, ex["crop"])[0, 0], np.array(ex["y"], float), atol=1e-13)
    np.testing.assert_allclose(oaa_ref.fft_conv_fwd(x, w, ex["crop"])[0, 0], np.array(ex["y"], float), atol=1e-12)


# ------------------------------------------------------------- 3-way equivalence
CASES = [(1, 1), (5, 1), (5, 2), (6, 3), (7, 3), (8, 4), (9, 5), (12, 5), (13, 7), (16, 8), (17, 8), (8, 8), (3, 5)]


@pytest.mark.parametrize("crop", CROPS)
@pytest.mark.parametrize("N,n", CASES)
@pytest.mark.parametrize("pow2", [False, True])
def test_oaa_equals_direct_equals_fftconv(N, n, crop, pow2):
    if crop == "valid" and n > N:
        pytest.skip("Valid needs n <= N")
    B, C, K = 2, 3, 2
    x, w = rnd(B, C, N, N), rnd(K, C, n, n)
    P = oaa_ref.next_pow2(2 * n - 1) if pow2 else None
    direct = oracle.conv_fwd(x, w, crop)
    oaa, imag = oaa_ref.oaa_conv_fwd(x, w, crop, P=P, return_imag=True)
    assert imag <= 1e-8 * max(1.0, np.abs(direct).max())        # SPEC.md:268 imaginary residue
    np.testing.assert_allclose(oaa, direct, rtol=0, atol=tol(C, n))
    np.testing.assert_allclose(oaa_ref.fft_conv_fwd(x, w, crop), direct, rtol=0, atol=tol(C, n))
    # numpy-FFT evaluation of the same OaA steps
    np.testing.assert_allclose(oaa_ref.oaa_conv_fwd(x, w, crop, P=P, use_numpy_fft=True), direct, atol=tol(C, n))


@pytest.mark.parametrize("crop", CROPS)
@pytest.mark.parametrize("N,n", [(6, 3), (9, 4), (11, 5), (16, 8), (8, 8), (7, 1), (10, 2)])
@pytest.mark.parametrize("pow2", [False, True])
def test_oaa_backward_equals_direct(N, n, crop, pow2):
    B, C, K = 2, 3, 2
    x, w = rnd(B, C, N, N), rnd(K, C, n, n)
    M = oaa_ref.out_size(N, n, crop)
    dy = rnd(B, K, M, M)
    P = oaa_ref.next_pow2(2 * n - 1) if pow2 else None
    np.testing.assert_allclose(oaa_ref.oaa_conv_bwd_data(dy, w, N, crop, P=P),
                               oracle.conv_bwd_data(dy, w, N, crop), atol=tol(K, n))
    np.testing.assert_allclose(oaa_ref.oaa_conv_bwd_filter(x, dy, n, crop, P=P),
                               oracle.conv_bwd_filter(x, dy, n, crop), atol=tol(B * 1.0, N))


@pytest.mark.parametrize("crop", CROPS)
def test_oaa_rectangular(crop):
    x, w = rnd(2, 2, 7, 10), rnd(3, 2, 2, 3)
    np.testing.assert_allclose(oaa_ref.oaa_conv_fwd(x, w, crop), oracle.conv_fwd(x, w, crop), atol=1e-11)
    M = oracle.conv_fwd(x, w, crop).shape[-2:]
    dy = rnd(2, 3, *M)
    np.testing.assert_allclose(oaa_ref.oaa_conv_bwd_data(dy, w, (7, 10), crop),
                               oracle.conv_bwd_data(dy, w, (7, 10), crop), atol=1e-11)
    np.testing.assert_allclose(oaa_ref.oaa_conv_bwd_filter(x, dy, (2, 3), crop),
                               oracle.conv_bwd_filter(x, dy, (2, 3), crop), atol=1e-11)


def test_aliasing_when_P_too_small():
    """P = 2n−2 wraps the (2n−1)-long block convolution: OaA then differs from the
    definition, so P ≥ 2n−1 is a real requirement, not a tuning knob."""
    x, w = rnd(1, 1, 16, 16), rnd(1, 1, 4, 4)
    bad = oaa_ref.oaa_conv_fwd(x, w, "full", P=2 * 4 - 2)
    assert np.abs(bad - oracle.conv_fwd(x, w, "full")).max() > 1e-3


def test_n_equals_N_single_block():
    """n = N gives one block at the same transform size as FFTconv."""
    x, w = rnd(1, 2, 8, 8), rnd(2, 2, 8, 8)
    assert oaa_ref.oaa_block_count(8, 8) == 1
    np.testing.assert_allclose(oaa_ref.oaa_conv_fwd(x, w, "full"), oaa_ref.fft_conv_fwd(x, w, "full"), atol=1e-11)


def test_n_one_is_scalar_multiply():
    """1×1 kernel → P = 1, each block a scalar multiply."""
    x, w = rnd(2, 3, 6, 6), rnd(4, 3, 1, 1)
    exp = np.einsum("kc,bcij->bkij", w[:, :, 0, 0], x)
    np.testing.assert_allclose(oaa_ref.oaa_conv_fwd(x, w, "full"), exp, atol=1e-14)


def test_complexity_numbers_paper():
    """for N=256, n=5: log2 N = 8 and log2 n ≈ 2.3 (the per-element factors
    of FFTconv and OaAconv), n² = 25 for spaceConv."""
    ex = GOLD["complexity"][0]
    assert ex["n"] ** 2 == ex["space"]
    assert math.log2(ex["N"]) == ex["fft"]
    assert round(math.log2(ex["n"]), 1) == ex["oaa"]


# -------------------------------------------------------------- overlap-and-save
@pytest.mark.parametrize("crop", CROPS)
@pytest.mark.parametrize("N,n", [(12, 3), (13, 4), (9, 5), (5, 5), (7, 1), (20, 8), (10, 2), (17, 7)])
def test_oas_equals_direct(N, n, crop):
    """Overlap-and-save (the variant the paper names beside OaA) reaches the
    linear convolution exactly: == the direct definition (scipy-pinned) for every crop."""
    if crop == "valid" and n > N:
        pytest.skip("Valid needs n <= N")
    x, w = rnd(2, 3, N, N), rnd(4, 3, n, n)
    np.testing.assert_allclose(oaa_ref.oas_conv_fwd(x, w, crop), oracle.conv_fwd(x, w, crop), atol=tol(3, n))
    # a larger (power-of-two) transform gives the identical result (reading R3)
    P = 1 << (2 * n - 1).bit_length() if n > 1 else 1
    np.testing.assert_allclose(oaa_ref.oas_conv_fwd(x, w, crop, P=P), oracle.conv_fwd(x, w, crop), atol=tol(3, n))


@pytest.mark.parametrize("n", [2, 3, 5, 8])
def test_oas_discarded_samples_are_aliased(n):
    """The first n−1 samples of each circular segment convolution wrap around: keeping
    them instead of the last n breaks the result (so step 4's discard is load-bearing),
    while n = 1 has nothing to discard."""
    x, w = rnd(1, 2, 3 * n + 1, 3 * n + 1), rnd(2, 2, n, n)
    bad = oaa_ref.oas_conv_fwd(x, w, "full", keep_aliased=True)
    assert np.abs(bad - oracle.conv_fwd(x, w, "full")).max() > 1e-3
    x1, w1 = rnd(1, 2, 6, 6), rnd(2, 2, 1, 1)
    np.testing.assert_allclose(oaa_ref.oas_conv_fwd(x1, w1, "full", keep_aliased=True),
                               oracle.conv_fwd(x1, w1, "full"), atol=1e-13)


def test_oas_delta_kernel_shift():
    """δ at (n−1, n−1) in Valid mode gives x[:M, :M] (a closed form)."""
    N, n = 11, 4
    x = rnd(1, 1, N, N)
    w = np.zeros((1, 1, n, n)); w[0, 0, n - 1, n - 1] = 1.0
    M = N - n + 1
    np.testing.assert_allclose(oaa_ref.oas_conv_fwd(x, w, "valid")[0, 0], x[0, 0, :M, :M], atol=1e-14)


# ------------------------------------------------------------- block size b != n (R18)
@pytest.mark.parametrize("crop", CROPS)
@pytest.mark.parametrize("N,n,b", [(20, 3, 13), (17, 5, 11), (14, 7, 9), (9, 3, 4), (11, 4, 12), (8, 2, 5),
                                   (23, 6, 10), (5, 3, 13)])
def test_oaa_block_size_b_ne_n_equals_direct(N, n, b, crop):
    """DESIGN.md R18: overlap-and-add with b×b blocks transformed at
    P = b + n − 1 is the same linear convolution as the definition, for all three passes
    (the forward block results are (b+n−1)² long and overlap by n−1; the weight gradient
    correlates b×b dy blocks with (b+n−1)² x-windows) -- including b > N (one block)."""
    if crop == "valid" and n > N:
        pytest.skip("Valid needs n <= N")
    B, C, K = 2, 2, 3
    x, w = rnd(B, C, N, N), rnd(K, C, n, n)
    M = oaa_ref.out_size(N, n, crop)
    dy = rnd(B, K, M, M)
    y, imag = oaa_ref.oaa_conv_fwd(x, w, crop, b=b, return_imag=True)
    assert imag <= 1e-8
    np.testing.assert_allclose(y, oracle.conv_fwd(x, w, crop), rtol=0, atol=tol(C, n))
    np.testing.assert_allclose(oaa_ref.oaa_conv_bwd_data(dy, w, N, crop, b=b),
                               oracle.conv_bwd_data(dy, w, N, crop), rtol=0, atol=tol(K, n))
    np.testing.assert_allclose(oaa_ref.oaa_conv_bwd_filter(x, dy, n, crop, b=b),
                               oracle.conv_bwd_filter(x, dy, n, crop), rtol=0, atol=tol(B * 1.0, N))


def test_block_size_aliasing_when_P_too_small():
    """With b×b blocks the block results are b + n − 1 long: P = b + n − 2 wraps them, so the
    product's P = 15 for b = 16 − n is the smallest exact grid."""
    x, w = rnd(1, 1, 26, 26), rnd(1, 1, 3, 3)
    bad = oaa_ref.oaa_conv_fwd(x, w, "full", P=13 + 3 - 2, b=13)
    assert np.abs(bad - oracle.conv_fwd(x, w, "full")).max() > 1e-3
    np.testing.assert_allclose(oaa_ref.oaa_conv_fwd(x, w, "full", P=15, b=13), oracle.conv_fwd(x, w, "full"),
                               atol=tol(1, 3))
