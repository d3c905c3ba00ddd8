"""GPU parity: the CUDA path (through the C ABI) vs the CPU float64 oracle.

Bar (BASELINE.json north_star): for every output tensor, rel-L2 = ‖out−ref‖₂/‖ref‖₂ ≤ 1e-5
and max|out−ref| ≤ 1e-4·max|ref|.  Small cases compare every element with the full
oracle; BASELINE's full-size configs compare seeded samples of outputs that the oracle
evaluates one by one (oracle.*_sample), plus the adjoint identity at full size.
"""
import itertools
import math

import numpy as np
import pytest
import torch

import oracle
import paper_1601_06815_b200 as oaa
from workloads import CONFIGS, SWEEP, make_inputs, out_size

pytestmark = pytest.mark.gpu

RTOL_L2 = 1e-5
RTOL_MAX = 1e-4
CROPS = ["full", "valid", "same"]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    torch.cuda.init()


def check(got, ref, what=""):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape, (what, got.shape, ref.shape)
    assert np.isfinite(got).all(), f"{what}: non-finite output"
    nref = np.linalg.norm(ref)
    err = np.linalg.norm(got - ref)
    mref = np.abs(ref).max() if ref.size else 0.0
    merr = np.abs(got - ref).max() if ref.size else 0.0
    if nref == 0:
        assert merr == 0.0, f"{what}: expected zeros, max err {merr}"
        return
    assert err <= RTOL_L2 * nref, f"{what}: rel-L2 {err / nref:.3e} > {RTOL_L2}"
    assert merr <= RTOL_MAX * mref, f"{what}: max-abs {merr:.3e} > {RTOL_MAX}·{mref:.3e}"


def run_all(d, N, n, crop):
    x = torch.from_numpy(d["x"]).cuda()
    w = torch.from_numpy(d["w"]).cuda()
    dy = torch.from_numpy(d["dy"]).cuda()
    y = oaa.conv_fwd(x, w, crop)
    dx = oaa.conv_bwd_data(dy, w, N, crop)
    dw = oaa.conv_bwd_filter(x, dy, n, crop)
    torch.cuda.synchronize()
    return y.cpu().numpy(), dx.cpu().numpy(), dw.cpu().numpy()


SMALL = [(N, n) for n in range(1, 9) for N in sorted({1, 2, n, n + 1, 2 * n - 1, 3 * n + 2, 17, 20})]


@pytest.mark.parametrize("crop", CROPS)
@pytest.mark.parametrize("N,n", SMALL)
def test_small_grid_all_passes(N, n, crop):
    if crop == "valid" and n > N:
        pytest.skip("Valid needs n <= N")
    for (B, C, K) in [(1, 1, 1), (2, 3, 2), (3, 2, 3)]:
        d = make_inputs(B, C, K, N, n, crop, seed=N * 100 + n * 7 + B)
        y, dx, dw = run_all(d, N, n, crop)
        check(y, oracle.conv_fwd(d["x"], d["w"], crop), f"fwd N={N} n={n} {crop} BCK={B,C,K}")
        check(dx, oracle.conv_bwd_data(d["dy"], d["w"], N, crop), f"bwd_data N={N} n={n} {crop}")
        check(dw, oracle.conv_bwd_filter(d["x"], d["dy"], n, crop), f"bwd_filter N={N} n={n} {crop}")


@pytest.mark.parametrize("crop", CROPS)
@pytest.mark.parametrize("B,C,K", [(2, 5, 3), (1, 4, 9), (2, 7, 6), (1, 1, 13)])
def test_channel_regimes(B, C, K, crop):
    """C ≤ 4 takes the input-stationary path, C > 4 the output-stationary chunked one;
    K > 4 / C > 4 exercise the chunk loops of bwd_data and bwd_filter."""
    N, n = 19, 4
    d = make_inputs(B, C, K, N, n, crop, seed=B * 31 + C * 7 + K)
    y, dx, dw = run_all(d, N, n, crop)
    check(y, oracle.conv_fwd(d["x"], d["w"], crop), "fwd")
    check(dx, oracle.conv_bwd_data(d["dy"], d["w"], N, crop), "bwd_data")
    check(dw, oracle.conv_bwd_filter(d["x"], d["dy"], n, crop), "bwd_filter")


@pytest.mark.parametrize("crop", CROPS)
@pytest.mark.parametrize("B,C,K,N,n", [(2, 16, 20, 17, 3), (1, 17, 33, 29, 5), (3, 24, 16, 20, 8),
                                       (2, 16, 16, 9, 1), (1, 20, 18, 40, 7), (2, 33, 17, 23, 2),
                                       (1, 16, 130, 12, 3), (1, 200, 16, 10, 5), (2, 32, 32, 32, 8),
                                       (2, 48, 96, 32, 8)])
def test_tensor_core_path(B, C, K, N, n, crop):
    """C ≥ 16 and K ≥ 16: fwd and bwd_data run tile spectra → tcgen05 bin GEMM (3×TF32)
    → walker (load mode); ragged 2C (K padding), ragged GEMM tiles, ragged spatial tails.
    2·Cout > 256 (K = 130 fwd, C = 200 bwd_data) takes the pre-split block-spectra GEMM
    (≥ 3 M tiles); the other cases split in the GEMM's converter warps.  (2, 32, 32, 32, 8) and
    (2, 48, 96, 32, 8) have whole walker chunks per tile row and 32-row output-channel groups,
    so their GEMM drains store Ŷ with TMA tensor stores (the other cases with st.global)."""
    if crop == "valid" and n > N:
        pytest.skip("Valid needs n <= N")
    d = make_inputs(B, C, K, N, n, crop, seed=B * 131 + C * 17 + K * 3 + n)
    y, dx, dw = run_all(d, N, n, crop)
    check(y, oracle.conv_fwd(d["x"], d["w"], crop), f"fwd tc {B,C,K,N,n}")
    check(dx, oracle.conv_bwd_data(d["dy"], d["w"], N, crop), f"bwd_data tc {B,C,K,N,n}")
    check(dw, oracle.conv_bwd_filter(d["x"], d["dy"], n, crop), "bwd_filter")


@pytest.mark.parametrize("crop", CROPS)
@pytest.mark.parametrize("B,C,K,N,n", [(2, 32, 16, 30, 7), (3, 16, 16, 30, 6), (1, 17, 40, 50, 7),
                                       (2, 40, 24, 70, 6), (1, 16, 33, 27, 7)])
def test_tensor_core_path_big_blocks(B, C, K, N, n, crop):
    """C, K >= 16 with n = 6, 7 and blocks b = 16 − n on the P = 15 grid (R18): tile
    spectra, realified weights, bin GEMM (120 bins) and the load walker of fwd / stand-alone
    bwd_data; every element of all three ops against the oracle, prepared spectra bitwise.
    (n ≤ 5 keeps b = n on this path.)"""
    assert oaa.block_size("fwd", C, K, N, n, crop) == 16 - n
    assert oaa.block_size("fwd", C, K, N, 5, crop) == 5
    d = make_inputs(B, C, K, N, n, crop, seed=B * 37 + C * 5 + K + N + n)
    y, dx, dw = run_all(d, N, n, crop)
    check(y, oracle.conv_fwd(d["x"], d["w"], crop), f"fwd tc b=16-n {B,C,K,N,n,crop}")
    check(dx, oracle.conv_bwd_data(d["dy"], d["w"], N, crop), f"bwd_data tc {B,C,K,N,n,crop}")
    check(dw, oracle.conv_bwd_filter(d["x"], d["dy"], n, crop), f"bwd_filter tc {B,C,K,N,n,crop}")
    x = torch.from_numpy(d["x"]).cuda(); w = torch.from_numpy(d["w"]).cuda()
    yp = oaa.PreparedWeights(w, N, "fwd", crop).fwd(x)
    torch.cuda.synchronize()
    assert torch.equal(yp.cpu(), torch.from_numpy(y))


@pytest.mark.parametrize("crop", ["valid", "same"])
@pytest.mark.parametrize("n", [3, 5, 8])
def test_largest_images(n, crop):
    """N = 250, near the v1 limit: 8 chunk warps in the walker / bwd_data kernels (n = 8),
    and the fallback engine where a tile row needs more than 8 chunk warps (n = 3)."""
    B, C, K, N = 2, 3, 9, 250
    d = make_inputs(B, C, K, N, n, crop, seed=250 + n)
    y, dx, dw = run_all(d, N, n, crop)
    check(y, oracle.conv_fwd(d["x"], d["w"], crop), f"fwd N=250 n={n} {crop}")
    check(dx, oracle.conv_bwd_data(d["dy"], d["w"], N, crop), f"bwd_data N=250 n={n} {crop}")
    check(dw, oracle.conv_bwd_filter(d["x"], d["dy"], n, crop), f"bwd_filter N=250 n={n} {crop}")


def _big_block_cases():
    # forward walker with blocks b = 16 − n (P = 15) for 3 <= n <= 7 once N >= 3b (or 2b with
    # little padding): N = 2b, the 3b threshold, one past it, ragged (the last block mostly
    # padding) and several chunks per tile row (stage B in two 32-column rounds when 4b > 32);
    # C = 1..4 register channels
    out = []
    for n in range(3, 8):
        b = 16 - n
        for i, N in enumerate(sorted({2 * b, 3 * b, 3 * b + 1, 4 * b - 1, 7 * b + 2, 100})):
            out.append((1 + i % 2, 1 + (n + i) % 4, 3 + 2 * i, N, n))
    return out


@pytest.mark.parametrize("crop", CROPS)
@pytest.mark.parametrize("B,C,K,N,n", _big_block_cases())
def test_walker_block_size_b_ne_n(B, C, K, N, n, crop):
    """SURVEY.md §8(f) NEXT-4 "block sizes b != n": the forward walker tiles the
    input, and bwd_data (C <= 4 output channels) tiles dy, into b×b blocks, b = 16 − n,
    transformed on the (b + n − 1)² = 15² grid; the results are the same linear convolutions
    (every element vs the direct oracle), and prepared spectra (their own P) give them
    bitwise."""
    assert oaa.block_size("fwd", C, K, N, n, crop) == 16 - n  # the larger blocks run
    d = make_inputs(B, C, K, N, n, crop, seed=N * 7 + n * 3 + C)
    x = torch.from_numpy(d["x"]).cuda()
    w = torch.from_numpy(d["w"]).cuda()
    dy = torch.from_numpy(d["dy"]).cuda()
    y = oaa.conv_fwd(x, w, crop)
    yp = oaa.PreparedWeights(w, N, "fwd", crop).fwd(x)
    dx = oaa.conv_bwd_data(dy, w, N, crop)
    dxp = oaa.PreparedWeights(w, N, "bwd_data", crop).bwd_data(dy)
    torch.cuda.synchronize()
    assert torch.equal(y, yp) and torch.equal(dx, dxp)
    check(y.cpu().numpy(), oracle.conv_fwd(d["x"], d["w"], crop), f"fwd b=16-n N={N} n={n} C={C} {crop}")
    check(dx.cpu().numpy(), oracle.conv_bwd_data(d["dy"], d["w"], N, crop), f"bwd_data b=16-n N={N} n={n} C={C} {crop}")


@pytest.mark.parametrize("crop", CROPS)
def test_config1_parity(crop):
    """BASELINE config 1: N=32, n=3, C=K=B=1, forward, vs CPU float64 direct."""
    c = CONFIGS["parity"]
    d = make_inputs(c.B, c.C, c.K, c.N, c.n, crop, seed=0)
    x = torch.from_numpy(d["x"]).cuda()
    w = torch.from_numpy(d["w"]).cuda()
    y = oaa.conv_fwd(x, w, crop).cpu().numpy()
    check(y, oracle.conv_fwd(d["x"], d["w"], crop), f"config1 {crop}")


def test_delta_kernel_and_zero():
    N, n = 23, 5
    x = torch.rand(2, 3, N, N, device="cuda") * 2 - 1
    w = torch.zeros(4, 3, n, n, device="cuda")
    assert oaa.conv_fwd(x, w, "valid").abs().max().item() == 0.0
    w[1, 2, 0, 0] = 1.0
    y = oaa.conv_fwd(x, w, "full")
    exp = torch.zeros(2, N + n - 1, N + n - 1, device="cuda")
    exp[:, :N, :N] = x[:, 2]
    assert (y[:, 1] - exp).abs().max().item() <= 1e-5
    dy = torch.zeros(2, 4, N - n + 1, N - n + 1, device="cuda")
    assert oaa.conv_bwd_data(dy, w, N, "valid").abs().max().item() == 0.0
    assert oaa.conv_bwd_filter(x, dy, n, "valid").abs().max().item() == 0.0


def test_batch_zero_is_noop_and_dw_zeroed():
    x = torch.empty(0, 3, 16, 16, device="cuda")
    w = torch.rand(4, 3, 3, 3, device="cuda")
    dy = torch.empty(0, 4, 14, 14, device="cuda")
    assert oaa.conv_fwd(x, w).shape == (0, 4, 14, 14)
    assert oaa.conv_bwd_data(dy, w, 16).shape == (0, 3, 16, 16)
    dw = torch.full((4, 3, 3, 3), 7.0, device="cuda")
    oaa.conv_bwd_filter(x, dy, 3, out=dw)
    assert dw.abs().max().item() == 0.0


def test_deterministic_and_stream_ordered():
    c = CONFIGS["headline"]
    d = make_inputs(4, c.C, c.K, c.N, c.n, "valid", seed=3)
    x = torch.from_numpy(d["x"]).cuda(); w = torch.from_numpy(d["w"]).cuda()
    dy = torch.from_numpy(d["dy"]).cuda()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        y1 = oaa.conv_fwd(x, w); dx1 = oaa.conv_bwd_data(dy, w, c.N); dw1 = oaa.conv_bwd_filter(x, dy, c.n)
        y2 = oaa.conv_fwd(x, w); dx2 = oaa.conv_bwd_data(dy, w, c.N); dw2 = oaa.conv_bwd_filter(x, dy, c.n)
    s.synchronize()
    assert torch.equal(y1, y2) and torch.equal(dx1, dx2) and torch.equal(dw1, dw2)


def test_concurrent_streams_match_sequential():
    """The three ops on three streams at once (the bench step runs bwd_filter beside
    bwd_data): every call gets its own workspace and the results are bitwise those of
    the sequential calls -- including the red.add overlap-add of bwd_data, whose two
    addends per element meet on an exact zero in either order."""
    c = CONFIGS["headline"]
    B = 6
    d = make_inputs(B, c.C, c.K, c.N, c.n, "valid", seed=17)
    x = torch.from_numpy(d["x"]).cuda(); w = torch.from_numpy(d["w"]).cuda()
    dy = torch.from_numpy(d["dy"]).cuda()
    y0 = oaa.conv_fwd(x, w); dx0 = oaa.conv_bwd_data(dy, w, c.N); dw0 = oaa.conv_bwd_filter(x, dy, c.n)
    torch.cuda.synchronize()
    s1, s2, s3 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(3):
        y = oaa.conv_fwd(x, w, stream=s1)
        dx = oaa.conv_bwd_data(dy, w, c.N, stream=s2)
        dw = oaa.conv_bwd_filter(x, dy, c.n, stream=s3)
        torch.cuda.synchronize()
        assert torch.equal(y, y0) and torch.equal(dx, dx0) and torch.equal(dw, dw0)


def test_outputs_fully_overwritten():
    N, n, crop = 30, 6, "same"
    d = make_inputs(2, 2, 3, N, n, crop, seed=11)
    x = torch.from_numpy(d["x"]).cuda(); w = torch.from_numpy(d["w"]).cuda()
    out = torch.full((2, 3, N, N), float("nan"), device="cuda")
    oaa.conv_fwd(x, w, crop, out=out)
    check(out.cpu().numpy(), oracle.conv_fwd(d["x"], d["w"], crop), "fwd into NaN buffer")


def test_autograd_module():
    N, n = 18, 3
    d = make_inputs(2, 3, 4, N, n, "valid", seed=5)
    layer = oaa.OaAConv2d(3, 4, n).cuda()
    with torch.no_grad():
        layer.weight.copy_(torch.from_numpy(d["w"]))
    x = torch.from_numpy(d["x"]).cuda().requires_grad_(True)
    y = layer(x)
    y.backward(torch.from_numpy(d["dy"]).cuda())
    check(y.detach().cpu().numpy(), oracle.conv_fwd(d["x"], d["w"], "valid"), "module fwd")
    check(x.grad.cpu().numpy(), oracle.conv_bwd_data(d["dy"], d["w"], N, "valid"), "module dx")
    check(layer.weight.grad.cpu().numpy(), oracle.conv_bwd_filter(d["x"], d["dy"], n, "valid"), "module dw")


# ----------------------------------------------------------- full-size, sampled
def _gpu_inputs(B, C, K, N, n, crop, seed):
    """Seeded synthetic inputs drawn on the device (uniform [-1,1), the SURVEY §8(d)
    recipe) -- for sizes where a CPU draw + copy would dominate the test time."""
    M = out_size(N, n, crop)
    g = torch.Generator(device="cuda")
    g.manual_seed(1000 + seed)
    x = torch.rand((B, C, N, N), generator=g, device="cuda") * 2 - 1
    w = torch.rand((K, C, n, n), generator=g, device="cuda") * 2 - 1
    dy = torch.rand((B, K, M, M), generator=g, device="cuda") * 2 - 1
    return x, w, dy


def _sample_idx(rng, shape, count, extra=()):
    idx = [tuple(int(rng.integers(0, s)) for s in shape) for _ in range(count)]
    # edges and corners of the spatial dims (ragged tails / tile seams)
    S1, S2 = shape[2], shape[3]
    for a, b in itertools.product([0, 1, S1 // 2, S1 - 2, S1 - 1], [0, 1, S2 // 2, S2 - 2, S2 - 1]):
        idx.append((int(rng.integers(0, shape[0])), int(rng.integers(0, shape[1])), max(0, a), max(0, b)))
    idx += list(extra)
    return np.array(idx, dtype=np.int64)


def _check_sampled(got_t, idx, ref, what):
    got = got_t[tuple(torch.from_numpy(idx[:, i]).to(got_t.device) for i in range(4))].double().cpu().numpy()
    # the sampled oracle values stand in for the full tensor's norm: compare per-sample
    # errors against the sampled reference scale (≥ the RMS of a dense sample)
    err = np.abs(got - ref)
    scale = np.sqrt(np.mean(ref ** 2))
    assert np.isfinite(got).all(), what
    assert np.sqrt(np.mean(err ** 2)) <= RTOL_L2 * scale * 1.0 + 1e-30, \
        f"{what}: sampled rel-L2 {np.sqrt(np.mean(err ** 2)) / scale:.3e}"
    assert err.max() <= RTOL_MAX * max(np.abs(ref).max(), scale), f"{what}: sampled max err {err.max():.3e}"


def _adjoint(y, dy, x, dx, w, dw):
    a = float((y.double() * dy.double()).sum())
    b = float((x.double() * dx.double()).sum())
    c = float((w.double() * dw.double()).sum())
    scale = math.sqrt(float((y.double() ** 2).sum()) * float((dy.double() ** 2).sum()))
    assert abs(a - b) <= 1e-5 * scale, (a, b, scale)
    assert abs(a - c) <= 1e-5 * scale, (a, c, scale)


def _full_size(cfg, crop="valid", n_samples=1500, n_dw=48, seed=0, sub_b=None):
    B, C, K, N, n = cfg.B, cfg.C, cfg.K, cfg.N, cfg.n
    x, w, dy = _gpu_inputs(B, C, K, N, n, crop, seed)
    y = oaa.conv_fwd(x, w, crop)
    dx = oaa.conv_bwd_data(dy, w, N, crop)
    dw = oaa.conv_bwd_filter(x, dy, n, crop)
    torch.cuda.synchronize()
    rng = np.random.default_rng(seed)
    # fwd / bwd_data: sampled images only need their own inputs on the host
    bsel = sorted(set(int(v) for v in rng.integers(0, B, size=sub_b or 4)) | {0, B - 1})
    xs = x[bsel].cpu().numpy(); ws_ = w.cpu().numpy(); dys = dy[bsel].cpu().numpy()
    M = out_size(N, n, crop)
    iy = _sample_idx(rng, (len(bsel), K, M, M), n_samples)
    ref = oracle.fwd_sample(xs, ws_, crop, iy)
    iy_g = iy.copy(); iy_g[:, 0] = np.array(bsel)[iy[:, 0]]
    _check_sampled(y, iy_g, ref, f"{cfg.name} fwd")
    ix = _sample_idx(rng, (len(bsel), C, N, N), n_samples)
    ref = oracle.bwd_data_sample(dys, ws_, N, crop, ix)
    ix_g = ix.copy(); ix_g[:, 0] = np.array(bsel)[ix[:, 0]]
    _check_sampled(dx, ix_g, ref, f"{cfg.name} bwd_data")
    # bwd_filter: each sampled dw element sums the whole batch
    kc = sorted(set((int(rng.integers(0, K)), int(rng.integers(0, C))) for _ in range(max(1, n_dw // (n * n)))))
    for (k, c) in kc:
        xk = x[:, c:c + 1].contiguous().cpu().numpy()
        dyk = dy[:, k:k + 1].contiguous().cpu().numpy()
        iw = np.array([(0, 0, u, v) for u in range(n) for v in range(n)], dtype=np.int64)
        ref = oracle.bwd_filter_sample(xk, dyk, n, crop, iw)
        got = dw[k, c].reshape(-1).double().cpu().numpy()
        err = np.linalg.norm(got - ref)
        assert err <= RTOL_L2 * np.linalg.norm(ref), f"{cfg.name} dw[{k},{c}] rel {err / np.linalg.norm(ref):.3e}"
    _adjoint(y, dy, x, dx, w, dw)


def test_host_pipeline_matches_device_calls():
    """pipeline.HostStep (chunked H2D/compute/D2H) gives the same results as the plain
    device calls, bitwise (same kernels, same per-image work)."""
    from paper_1601_06815_b200.pipeline import HostStep
    B, C, K, N, n, crop = 6, 3, 5, 30, 5, "valid"
    d = make_inputs(B, C, K, N, n, crop, seed=13)
    hx = torch.from_numpy(d["x"]).pin_memory(); hw = torch.from_numpy(d["w"]).pin_memory()
    hdy = torch.from_numpy(d["dy"]).pin_memory()
    M = out_size(N, n, crop)
    hy = torch.empty((B, K, M, M)).pin_memory(); hdx = torch.empty((B, C, N, N)).pin_memory()
    hdw = torch.empty((K, C, n, n)).pin_memory()
    hs = HostStep(B, C, K, N, n, crop, chunks=3)
    hs(hx, hw, hdy, hy, hdx, hdw)
    torch.cuda.synchronize()
    x, w, dy = hx.cuda(), hw.cuda(), hdy.cuda()
    assert torch.equal(hy, oaa.conv_fwd(x, w, crop).cpu())
    assert torch.equal(hdx, oaa.conv_bwd_data(dy, w, N, crop).cpu())
    assert torch.equal(hdw, oaa.conv_bwd_filter(x, dy, n, crop).cpu())


@pytest.mark.parametrize("F,M,N,Kd", [(1, 128, 128, 32), (3, 256, 384, 192), (2, 200, 130, 68), (5, 512, 256, 128),
                                      (3, 300, 700, 50), (1, 16, 1000, 7), (2, 130, 257, 96)])
def test_tcgen05_bin_gemm_3xtf32(F, M, N, Kd):
    """The tensor-core contraction kernel alone vs a float64 matmul: fp32-level accuracy
    (3×TF32), ragged M/N/K tails."""
    g = torch.Generator(device="cuda").manual_seed(F * 1000 + M + N + Kd)
    A = torch.rand((F, M, Kd), generator=g, device="cuda") * 2 - 1
    B = torch.rand((F, N, Kd), generator=g, device="cuda") * 2 - 1
    D = oaa.debug_bin_gemm(A, B)
    ref = torch.matmul(A.double(), B.double().transpose(1, 2))
    check(D.cpu().numpy(), ref.cpu().numpy(), "bin_gemm")


# ----------------------------------------------------------- overlap-and-save forward
@pytest.mark.parametrize("crop", CROPS)
@pytest.mark.parametrize("N,n", [(N, n) for n in range(1, 9) for N in sorted({n, n + 1, 2 * n - 1, 3 * n + 2, 20, 33})])
def test_oas_forward_small_grid(N, n, crop):
    """NEXT-2: conv_fwd_oas == the direct oracle, every element, all crops,
    ragged output tiles, C ≤ 4 (the SIMT walker family)."""
    if crop == "valid" and n > N:
        pytest.skip("Valid needs n <= N")
    for (B, C, K) in [(1, 1, 1), (2, 3, 5), (3, 4, 9)]:
        d = make_inputs(B, C, K, N, n, crop, seed=N * 13 + n * 5 + B)
        x = torch.from_numpy(d["x"]).cuda()
        w = torch.from_numpy(d["w"]).cuda()
        y = oaa.conv_fwd_oas(x, w, crop)
        torch.cuda.synchronize()
        check(y.cpu().numpy(), oracle.conv_fwd(d["x"], d["w"], crop), f"oas N={N} n={n} {crop} BCK={B,C,K}")


@pytest.mark.parametrize("crop", CROPS)
@pytest.mark.parametrize("B,C,K,N,n", [(2, 16, 20, 17, 3), (1, 17, 33, 29, 5), (3, 24, 16, 20, 8),
                                       (2, 32, 32, 32, 8), (1, 20, 18, 40, 7), (2, 16, 16, 9, 1)])
def test_oas_tensor_core_path(B, C, K, N, n, crop):
    """Overlap-and-save for C, K ≥ 16: x-window spectra of the output tiles →
    tcgen05 bin GEMM → walker in load + overlap-and-save mode; every element vs the oracle."""
    if crop == "valid" and n > N:
        pytest.skip("Valid needs n <= N")
    d = make_inputs(B, C, K, N, n, crop, seed=B * 31 + C + K * 7 + N + n)
    x = torch.from_numpy(d["x"]).cuda(); w = torch.from_numpy(d["w"]).cuda()
    y = oaa.conv_fwd_oas(x, w, crop)
    torch.cuda.synchronize()
    check(y.cpu().numpy(), oracle.conv_fwd(d["x"], d["w"], crop), f"oas tc {B,C,K,N,n,crop}")


def test_oas_matches_oaa_and_rejects_large_C():
    d = make_inputs(2, 3, 64, 60, 8, "valid", seed=5)
    x = torch.from_numpy(d["x"]).cuda(); w = torch.from_numpy(d["w"]).cuda()
    a = oaa.conv_fwd_oas(x, w); b = oaa.conv_fwd(x, w)
    assert (a - b).abs().max().item() <= 1e-4 * b.abs().max().item()
    with pytest.raises(ValueError):
        oaa.conv_fwd_oas(torch.zeros(1, 5, 16, 16, device="cuda"), torch.zeros(2, 5, 3, 3, device="cuda"))


# ------------------------------------------------------ prepared (cached) weight spectra
@pytest.mark.parametrize("B,C,K,N,n,crop", [(2, 3, 8, 40, 8, "valid"), (2, 3, 5, 23, 5, "same"),
                                            (1, 6, 7, 19, 4, "full"), (2, 16, 20, 17, 3, "same"),
                                            (2, 24, 16, 20, 8, "valid"), (1, 2, 3, 250, 3, "valid")])
def test_prepared_weight_spectra_bitwise(B, C, K, N, n, crop):
    """NEXT-4: spectra prepared once give bitwise the unprepared results,
    for every kernel family (walker, bwd_data, flag engine, tensor-core path), and the
    prepared buffer is read-only across many calls."""
    d = make_inputs(B, C, K, N, n, crop, seed=B + C + K + N + n)
    x = torch.from_numpy(d["x"]).cuda(); w = torch.from_numpy(d["w"]).cuda()
    dy = torch.from_numpy(d["dy"]).cuda()
    pf = oaa.PreparedWeights(w, N, "fwd", crop)
    pb = oaa.PreparedWeights(w, N, "bwd_data", crop)
    snap_f, snap_b = pf.spec.clone(), pb.spec.clone()
    y0, dx0 = oaa.conv_fwd(x, w, crop), oaa.conv_bwd_data(dy, w, N, crop)
    for _ in range(2):
        assert torch.equal(pf.fwd(x), y0)
        assert torch.equal(pb.bwd_data(dy), dx0)
    torch.cuda.synchronize()
    assert torch.equal(pf.spec, snap_f) and torch.equal(pb.spec, snap_b)
    check(y0.cpu().numpy(), oracle.conv_fwd(d["x"], d["w"], crop), "prepared fwd")
    with pytest.raises(ValueError):
        pf.bwd_data(dy)


# ------------------------------------------------------------------ fused backward
@pytest.mark.parametrize("B,C,K,N,n,crop", [(2, 3, 8, 40, 8, "valid"), (3, 2, 5, 23, 5, "full"),
                                            (2, 16, 20, 17, 3, "same"), (3, 24, 16, 20, 8, "valid"),
                                            (2, 33, 17, 23, 2, "full"), (1, 200, 16, 10, 5, "same"),
                                            (5, 17, 33, 29, 5, "valid"),
                                            # tensor-core fused backward: ragged bt tails, 1-2
                                            # weight-gradient M tiles, split-K, several batch chunks
                                            (2, 16, 32, 17, 3, "same"), (2, 64, 128, 20, 8, "valid"),
                                            (1, 48, 64, 25, 5, "full"), (3, 32, 96, 14, 4, "valid"),
                                            (2, 64, 256, 12, 7, "same"), (9, 16, 32, 40, 6, "valid")])
def test_fused_backward(B, C, K, N, n, crop):
    """NEXT-1: oaa_conv_bwd gives dx bitwise equal to oaa_conv_bwd_data when
    both tile dy alike (a stand-alone bwd_data with blocks b = 16 − n, R18, rounds
    differently: then both are held to the oracle) and dw within the bar of the oracle (on
    the tensor-core path it shares the dy spectra between both GEMMs)."""
    d = make_inputs(B, C, K, N, n, crop, seed=7 * B + C + K + N + n)
    x = torch.from_numpy(d["x"]).cuda(); w = torch.from_numpy(d["w"]).cuda()
    dy = torch.from_numpy(d["dy"]).cuda()
    dx, dw = oaa.conv_bwd(x, dy, w, crop)
    dx1 = oaa.conv_bwd_data(dy, w, N, crop)
    torch.cuda.synchronize()
    if oaa.block_size("bwd_data", C, K, N, n, crop) == n:
        assert torch.equal(dx, dx1)
    else:
        check(dx1.cpu().numpy(), oracle.conv_bwd_data(d["dy"], d["w"], N, crop), "stand-alone dx (b != n)")
    check(dx.cpu().numpy(), oracle.conv_bwd_data(d["dy"], d["w"], N, crop), "fused dx")
    check(dw.cpu().numpy(), oracle.conv_bwd_filter(d["x"], d["dy"], n, crop), "fused dw")
    dx2, dw2 = oaa.conv_bwd(x, dy, w, crop)
    assert torch.equal(dx2, dx) and torch.equal(dw2, dw)  # deterministic


@pytest.mark.parametrize("B,N,n,crop", [(85, 60, 8, "valid"), (75, 64, 8, "same"), (40, 120, 8, "valid"),
                                        (97, 45, 5, "full")])
def test_bwd_data_several_pairs_per_cta(B, N, n, crop):
    """Narrow images: bwd_data puts several (image, tile row) pairs in one CTA (8 compute
    warps sharing one kernel-spectrum ring); B·T′ is chosen so that the pairs
    per CTA is 2-4 and the last CTA is ragged.  dx of every element against the oracle, and
    the fused backward's dx bitwise equal to it."""
    C, K = 3, 64
    d = make_inputs(B, C, K, N, n, crop, seed=B + N + n)
    w = torch.from_numpy(d["w"]).cuda()
    dy = torch.from_numpy(d["dy"]).cuda()
    x = torch.from_numpy(d["x"]).cuda()
    dx = oaa.conv_bwd_data(dy, w, N, crop)
    dxf, dwf = oaa.conv_bwd(x, dy, w, crop)
    torch.cuda.synchronize()
    check(dx.cpu().numpy(), oracle.conv_bwd_data(d["dy"], d["w"], N, crop), "bwd_data")
    assert torch.equal(dx, dxf)
    check(dwf.cpu().numpy(), oracle.conv_bwd_filter(d["x"], d["dy"], n, crop), "fused dw")


def test_cuda_graph_capture_replays_bitwise():
    """The library only enqueues kernels, memsets and attribute calls on the caller's
    stream (no allocation, no synchronisation; include/oaa.h), so a whole step can be
    captured into a CUDA graph and replayed -- the launch-latency remedy for small
    layers.  Replays give bitwise the eager results, on both kernel families."""
    for (B, C, K, N, n, crop) in [(4, 3, 16, 32, 5, "valid"), (2, 16, 20, 17, 3, "same")]:
        d = make_inputs(B, C, K, N, n, crop, seed=99)
        x = torch.from_numpy(d["x"]).cuda(); w = torch.from_numpy(d["w"]).cuda()
        dy = torch.from_numpy(d["dy"]).cuda()
        M = out_size(N, n, crop)
        y = torch.empty((B, K, M, M), device="cuda"); dx = torch.empty_like(x); dw = torch.empty_like(w)
        s = torch.cuda.Stream()

        def step():
            oaa.conv_fwd(x, w, crop, out=y, stream=s)
            oaa.conv_bwd(x, dy, w, crop, dx=dx, dw=dw, stream=s)

        with torch.cuda.stream(s):  # warm-up: workspaces allocated, kernels loaded
            step()
        torch.cuda.synchronize()
        y0, dx0, dw0 = y.clone(), dx.clone(), dw.clone()
        y.zero_(); dx.zero_(); dw.zero_()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            step()
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        assert torch.equal(y, y0) and torch.equal(dx, dx0) and torch.equal(dw, dw0)


def _random_shapes(count, seed):
    """Seeded random layer shapes across the three kernel families (C ≤ 4 SIMT kernels,
    5 ≤ C ≤ 15 first-generation engine, C, K ≥ 16 tensor-core path), all n and crops."""
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < count:
        fam = len(out) % 3
        n = int(rng.integers(1, 9))
        N = int(rng.integers(max(1, n), 48))
        crop = CROPS[int(rng.integers(0, 3))]
        B = int(rng.integers(1, 4))
        if fam == 0:
            C, K = int(rng.integers(1, 5)), int(rng.integers(1, 40))
        elif fam == 1:
            C, K = int(rng.integers(5, 16)), int(rng.integers(1, 12))
        else:
            C, K = int(rng.integers(16, 48)), int(rng.integers(16, 48))
        out.append((B, C, K, N, n, crop))
    return out


@pytest.mark.parametrize("B,C,K,N,n,crop", _random_shapes(60, 2026))
def test_random_shapes_all_ops(B, C, K, N, n, crop):
    """Seeded random shapes (every family, n, crop, ragged sizes): fwd, bwd_data, bwd_filter,
    the fused backward (dx bitwise equal to bwd_data) and, where supported, overlap-and-save —
    every element against the oracle."""
    d = make_inputs(B, C, K, N, n, crop, seed=B * 7 + C * 11 + K * 13 + N * 17 + n)
    y, dx, dw = run_all(d, N, n, crop)
    check(y, oracle.conv_fwd(d["x"], d["w"], crop), f"fwd {B,C,K,N,n,crop}")
    ref_dx = oracle.conv_bwd_data(d["dy"], d["w"], N, crop)
    ref_dw = oracle.conv_bwd_filter(d["x"], d["dy"], n, crop)
    check(dx, ref_dx, f"bwd_data {B,C,K,N,n,crop}")
    check(dw, ref_dw, f"bwd_filter {B,C,K,N,n,crop}")
    x = torch.from_numpy(d["x"]).cuda(); w = torch.from_numpy(d["w"]).cuda()
    dy = torch.from_numpy(d["dy"]).cuda()
    dxf, dwf = oaa.conv_bwd(x, dy, w, crop)
    torch.cuda.synchronize()
    check(dxf.cpu().numpy(), ref_dx, "fused dx")
    check(dwf.cpu().numpy(), ref_dw, "fused dw")
    if C <= 4 or (C >= 16 and K >= 16):
        yo = oaa.conv_fwd_oas(x, w, crop)
        torch.cuda.synchronize()
        check(yo.cpu().numpy(), oracle.conv_fwd(d["x"], d["w"], crop), "oas")


def _random_large_shapes(count, seed):
    """Seeded random large images (N up to the 256-column limit): many tile rows, up to 8
    chunk warps, both SIMT and tensor-core families."""
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < count:
        n = int(rng.integers(2, 9))
        N = int(rng.integers(100, 251))
        crop = CROPS[int(rng.integers(0, 3))]
        if max(-(-N // n) * n, N + n - 1 if crop == "full" else N) > 256:
            continue
        if len(out) % 2 == 0:
            B, C, K = int(rng.integers(1, 3)), int(rng.integers(1, 5)), int(rng.integers(1, 12))
        else:
            B, C, K = 1, int(rng.integers(16, 24)), int(rng.integers(16, 24))
        out.append((B, C, K, N, n, crop))
    return out


@pytest.mark.parametrize("B,C,K,N,n,crop", _random_large_shapes(30, 77))
def test_random_large_shapes(B, C, K, N, n, crop):
    d = make_inputs(B, C, K, N, n, crop, seed=B + C * 3 + K * 5 + N + n)
    y, dx, dw = run_all(d, N, n, crop)
    check(y, oracle.conv_fwd(d["x"], d["w"], crop), f"fwd {B,C,K,N,n,crop}")
    check(dx, oracle.conv_bwd_data(d["dy"], d["w"], N, crop), f"bwd_data {B,C,K,N,n,crop}")
    check(dw, oracle.conv_bwd_filter(d["x"], d["dy"], n, crop), f"bwd_filter {B,C,K,N,n,crop}")
