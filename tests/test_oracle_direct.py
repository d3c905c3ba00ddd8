"""Pins for the DIRECT fp64 oracle (oracle/oracle.c) against things other than itself.

  * scipy.signal.convolve2d (textbook library routine) for every crop, C=K=B=1 and
    channel sums ("each channel of each kernel is convolved with the
    respective channel"; SPEC.md:334 channel additivity);
  * torch.nn.functional.conv2d (correlation => flipped kernel) and its autograd for
    bwd_data / bwd_filter;
  * SPEC's worked examples (tests/golden, cited per entry);
  * delta-kernel identities with exactly known outputs;
  * the adjoint (dot-product) identity tying both gradients to the forward;
  * central finite differences;
  * linearity, zero annihilation, flip commutation.
"""
import itertools
import json
import os

import numpy as np
import pytest
import scipy.signal
import torch

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_worked_examples.json")))
CROPS = ["full", "valid", "same"]
RNG = np.random.default_rng(1234)


def rnd(*shape):
    return RNG.uniform(-1, 1, size=shape)


@pytest.mark.parametrize("crop", CROPS)
@pytest.mark.parametrize("N,n", [(1, 1), (4, 1), (5, 2), (6, 3), (7, 4), (8, 8), (9, 5), (3, 2)])
def test_fwd_matches_scipy_single_channel(N, n, crop):
    if crop == "valid" and n > N:
        pytest.skip("Valid needs n <= N")
    x, w = rnd(1, 1, N, N), rnd(1, 1, n, n)
    y = oracle.conv_fwd(x, w, crop)
    ref = scipy.signal.convolve2d(x[0, 0], w[0, 0], mode=crop)
    np.testing.assert_allclose(y[0, 0], ref, rtol=0, atol=1e-13)


@pytest.mark.parametrize("crop", CROPS)
def test_fwd_rectangular_matches_scipy(crop):
    x, w = rnd(1, 1, 5, 9), rnd(1, 1, 2, 3)
    y = oracle.conv_fwd(x, w, crop)
    np.testing.assert_allclose(y[0, 0], scipy.signal.convolve2d(x[0, 0], w[0, 0], mode=crop), atol=1e-13)


@pytest.mark.parametrize("crop", CROPS)
def test_fwd_multichannel_is_sum_of_scipy(crop):
    B, C, K, N, n = 2, 3, 4, 9, 3
    x, w = rnd(B, C, N, N), rnd(K, C, n, n)
    y = oracle.conv_fwd(x, w, crop)
    for b, k in itertools.product(range(B), range(K)):
        ref = sum(scipy.signal.convolve2d(x[b, c], w[k, c], mode=crop) for c in range(C))
        np.testing.assert_allclose(y[b, k], ref, atol=1e-12)


def _torch_layer(x, w, crop):
    """torch conv2d is a correlation: convolution = conv2d with the 180°-flipped kernel.
    Crops are built from Full (padding n−1) + slicing, so even-n Same matches scipy
    (reading R6)."""
    n = w.shape[-1]
    xt = torch.tensor(x, dtype=torch.float64, requires_grad=True)
    wt = torch.tensor(w, dtype=torch.float64, requires_grad=True)
    full = torch.nn.functional.conv2d(xt, torch.flip(wt, dims=(-2, -1)), padding=n - 1)
    N = x.shape[-1]
    o = {"full": 0, "valid": n - 1, "same": (n - 1) // 2}[crop]
    M = {"full": N + n - 1, "valid": N - n + 1, "same": N}[crop]
    return xt, wt, full[:, :, o:o + M, o:o + M]


@pytest.mark.parametrize("crop", CROPS)
@pytest.mark.parametrize("N,n", [(6, 3), (7, 4), (8, 8), (10, 5), (5, 1), (9, 2)])
def test_all_three_passes_match_torch_autograd(N, n, crop):
    B, C, K = 2, 3, 2
    x, w = rnd(B, C, N, N), rnd(K, C, n, n)
    xt, wt, yt = _torch_layer(x, w, crop)
    dy = rnd(*yt.shape)
    yt.backward(torch.tensor(dy))
    np.testing.assert_allclose(oracle.conv_fwd(x, w, crop), yt.detach().numpy(), atol=1e-12)
    np.testing.assert_allclose(oracle.conv_bwd_data(dy, w, N, crop), xt.grad.numpy(), atol=1e-12)
    np.testing.assert_allclose(oracle.conv_bwd_filter(x, dy, n, crop), wt.grad.numpy(), atol=1e-12)


@pytest.mark.parametrize("ex", GOLD["conv"], ids=lambda e: e["cite"][:12])
def test_spec_worked_examples(ex):
    x = np.array(ex["x"], dtype=np.float64)[None, None]
    w = np.array(ex["w"], dtype=np.float64)[None, None]
    y = oracle.conv_fwd(x, w, ex["crop"])
    np.testing.assert_array_equal(y[0, 0], np.array(ex["y"], dtype=np.float64))


@pytest.mark.parametrize("N,n", [(7, 3), (8, 4), (6, 1), (9, 8)])
def test_delta_kernel_identities(N, n):
    """δ at (0,0): Full = zero-padded x; Valid = x[n−1:, n−1:]; Same = x shifted
    up-left by floor((n−1)/2) with zero fill.  δ at (n−1,n−1): Valid = x[:M,:M]."""
    x = rnd(1, 1, N, N)
    d0 = np.zeros((1, 1, n, n)); d0[0, 0, 0, 0] = 1
    full = oracle.conv_fwd(x, d0, "full")[0, 0]
    exp = np.zeros((N + n - 1, N + n - 1)); exp[:N, :N] = x[0, 0]
    np.testing.assert_array_equal(full, exp)
    np.testing.assert_array_equal(oracle.conv_fwd(x, d0, "valid")[0, 0], x[0, 0, n - 1:, n - 1:])
    s = (n - 1) // 2
    same = np.zeros((N, N)); same[:N - s, :N - s] = x[0, 0, s:, s:]
    np.testing.assert_array_equal(oracle.conv_fwd(x, d0, "same")[0, 0], same)
    dl = np.zeros((1, 1, n, n)); dl[0, 0, n - 1, n - 1] = 1
    M = N - n + 1
    np.testing.assert_array_equal(oracle.conv_fwd(x, dl, "valid")[0, 0], x[0, 0, :M, :M])


@pytest.mark.parametrize("crop", CROPS)
@pytest.mark.parametrize("N,n", [(7, 3), (8, 4), (5, 5)])
def test_adjoint_identity(N, n, crop):
    """<fwd(x,w), dy> = <x, bwd_data(dy,w)> = <w, bwd_filter(x,dy)>."""
    B, C, K = 2, 2, 3
    x, w = rnd(B, C, N, N), rnd(K, C, n, n)
    y = oracle.conv_fwd(x, w, crop)
    dy = rnd(*y.shape)
    a = np.vdot(y, dy)
    b = np.vdot(x, oracle.conv_bwd_data(dy, w, N, crop))
    c = np.vdot(w, oracle.conv_bwd_filter(x, dy, n, crop))
    assert abs(a - b) <= 1e-12 * max(1.0, abs(a))
    assert abs(a - c) <= 1e-12 * max(1.0, abs(a))


@pytest.mark.parametrize("crop", CROPS)
def test_finite_differences(crop):
    """Central differences of L = Σ dy ⊙ fwd(x, w), step 1e−5."""
    B, C, K, N, n = 1, 2, 2, 6, 3
    x, w = rnd(B, C, N, N), rnd(K, C, n, n)
    dy = rnd(*oracle.conv_fwd(x, w, crop).shape)
    L = lambda xx, ww: float(np.vdot(oracle.conv_fwd(xx, ww, crop), dy))
    gx = oracle.conv_bwd_data(dy, w, N, crop)
    gw = oracle.conv_bwd_filter(x, dy, n, crop)
    h = 1e-5
    for idx in [(0, 0, 0, 0), (0, 1, 2, 3), (0, 0, 5, 5), (0, 1, 3, 0)]:
        xp, xm = x.copy(), x.copy(); xp[idx] += h; xm[idx] -= h
        fd = (L(xp, w) - L(xm, w)) / (2 * h)
        assert abs(fd - gx[idx]) <= 1e-5 * max(1.0, abs(gx[idx]))
    for idx in [(0, 0, 0, 0), (1, 1, 2, 1), (0, 1, 1, 2)]:
        wp, wm = w.copy(), w.copy(); wp[idx] += h; wm[idx] -= h
        fd = (L(x, wp) - L(x, wm)) / (2 * h)
        assert abs(fd - gw[idx]) <= 1e-5 * max(1.0, abs(gw[idx]))


def test_linearity_zero_and_flip():
    B, C, K, N, n = 1, 2, 2, 7, 3
    x, w1, w2 = rnd(B, C, N, N), rnd(K, C, n, n), rnd(K, C, n, n)
    a, b = 0.7, -1.3
    np.testing.assert_allclose(oracle.conv_fwd(x, a * w1 + b * w2, "full"),
                               a * oracle.conv_fwd(x, w1, "full") + b * oracle.conv_fwd(x, w2, "full"), atol=1e-12)
    assert not oracle.conv_fwd(x, np.zeros_like(w1), "valid").any()
    dyz = np.zeros((B, K, N - n + 1, N - n + 1))
    assert not oracle.conv_bwd_data(dyz, w1, N, "valid").any()
    assert not oracle.conv_bwd_filter(x, dyz, n, "valid").any()
    # flip commutation, single channel, Full
    x1, k1 = x[:, :1], w1[:1, :1]
    lhs = oracle.conv_fwd(x1[..., ::-1, ::-1], k1[..., ::-1, ::-1], "full")
    np.testing.assert_allclose(lhs, oracle.conv_fwd(x1, k1, "full")[..., ::-1, ::-1], atol=1e-13)


def test_channel_cancellation():
    """channel2 = −channel1 with equal kernels across channels → zero."""
    x = rnd(1, 1, 8, 8)
    x2 = np.concatenate([x, -x], axis=1)
    w = np.repeat(rnd(2, 1, 3, 3), 2, axis=1)
    assert np.abs(oracle.conv_fwd(x2, w, "valid")).max() <= 1e-14  # exact up to rounding order


def test_sampled_entry_points_match_full():
    from workloads import make_inputs
    for crop in CROPS:
        d = make_inputs(3, 2, 4, 11, 4, crop, seed=5)
        x, w, dy = d["x"], d["w"], d["dy"]
        y = oracle.conv_fwd(x, w, crop)
        dx = oracle.conv_bwd_data(dy, w, 11, crop)
        dw = oracle.conv_bwd_filter(x, dy, 4, crop)
        ii = np.stack(np.meshgrid(*[np.arange(s) for s in y.shape], indexing="ij"), -1).reshape(-1, 4)
        np.testing.assert_allclose(oracle.fwd_sample(x, w, crop, ii), y.reshape(-1), atol=1e-12)
        ii = np.stack(np.meshgrid(*[np.arange(s) for s in dx.shape], indexing="ij"), -1).reshape(-1, 4)
        np.testing.assert_allclose(oracle.bwd_data_sample(dy, w, 11, crop, ii), dx.reshape(-1), atol=1e-12)
        ii = np.stack(np.meshgrid(*[np.arange(s) for s in dw.shape], indexing="ij"), -1).reshape(-1, 4)
        np.testing.assert_allclose(oracle.bwd_filter_sample(x, dy, 4, crop, ii), dw.reshape(-1), atol=1e-12)
        y2, dx2, dw2 = oracle.step_f32(x, w, dy, crop)
        np.testing.assert_allclose(y2, y, atol=1e-12)
        np.testing.assert_allclose(dx2, dx, atol=1e-12)
        np.testing.assert_allclose(dw2, dw, atol=1e-12)


def test_sample_rejects_out_of_range():
    x = np.zeros((1, 1, 5, 5), np.float32); w = np.zeros((1, 1, 3, 3), np.float32)
    with pytest.raises(ValueError):
        oracle.fwd_sample(x, w, "valid", np.array([[0, 0, 3, 0]]))  # M = 3 -> i=3 invalid


def test_thread_count_invariance():
    from workloads import make_inputs
    d = make_inputs(2, 3, 5, 13, 5, "same", seed=9)
    a = oracle.conv_fwd(d["x"], d["w"], "same", nthreads=1)
    b = oracle.conv_fwd(d["x"], d["w"], "same", nthreads=4)
    np.testing.assert_array_equal(a, b)
