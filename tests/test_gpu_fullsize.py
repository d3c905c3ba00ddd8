"""Full-size GPU parity: every element of y, dx and dw at BASELINE.json's full configs,
in the launch configuration bench.py times, against the CPU float64 oracle.

Bar (BASELINE.json north_star): per output tensor, rel-L2 = ‖out−ref‖₂/‖ref‖₂ ≤ 1e-5 and
max|out−ref| ≤ 1e-4·max|ref|, both over the WHOLE tensor.  The oracle (oracle/oracle.c,
the direct definitions of SURVEY.md §8(c) items 1-3) runs on the host cores over chunks of
images; dw is a sum over the batch, so its chunks are summed in fp64 (the definition's
own sum, split).  Where the whole oracle is too slow (configs[4], 148 GFLOP per image)
the check covers whole images (every element of their y and dx), stratified dw elements
(every output channel k, every input channel c), and the sum-over-shards identity of dw.
Inputs: seeded uniform [-1, 1) drawn on the device (copying 1.5 GB
through the host would dominate), the same fp32 values handed to the oracle.
"""
import math

import numpy as np
import pytest
import torch

import oracle
import paper_1601_06815_b200 as oaa
from workloads import CONFIGS, SWEEP, Workload, out_size

pytestmark = pytest.mark.gpu

RTOL_L2 = 1e-5
RTOL_MAX = 1e-4


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    torch.cuda.init()


class Err:
    """Running ‖got−ref‖², ‖ref‖², max|got−ref|, max|ref| over chunks of a tensor."""

    def __init__(self, what):
        self.what, self.e2, self.r2, self.emax, self.rmax, self.n = what, 0.0, 0.0, 0.0, 0.0, 0

    def add(self, got, ref):
        got = np.asarray(got, dtype=np.float64)
        ref = np.asarray(ref, dtype=np.float64)
        assert got.shape == ref.shape, (self.what, got.shape, ref.shape)
        assert np.isfinite(got).all(), f"{self.what}: non-finite output"
        d = got - ref
        self.e2 += float(np.vdot(d, d))
        self.r2 += float(np.vdot(ref, ref))
        self.emax = max(self.emax, float(np.abs(d).max()) if d.size else 0.0)
        self.rmax = max(self.rmax, float(np.abs(ref).max()) if ref.size else 0.0)
        self.n += ref.size

    def check(self):
        rel = math.sqrt(self.e2 / self.r2) if self.r2 > 0 else 0.0
        assert self.n > 0, self.what
        assert rel <= RTOL_L2, f"{self.what}: rel-L2 {rel:.3e} > {RTOL_L2} over {self.n} elements"
        assert self.emax <= RTOL_MAX * self.rmax, \
            f"{self.what}: max-abs {self.emax:.3e} > {RTOL_MAX}·{self.rmax:.3e}"
        return rel


def gpu_inputs(B, C, K, N, n, crop, seed):
    M = out_size(N, n, crop)
    g = torch.Generator(device="cuda")
    g.manual_seed(1000 + seed)
    x = torch.rand((B, C, N, N), generator=g, device="cuda").mul_(2).sub_(1)
    w = torch.rand((K, C, n, n), generator=g, device="cuda").mul_(2).sub_(1)
    dy = torch.rand((B, K, M, M), generator=g, device="cuda").mul_(2).sub_(1)
    return x, w, dy


def run_ops(x, w, dy, N, n, crop):
    y = oaa.conv_fwd(x, w, crop)
    dx = oaa.conv_bwd_data(dy, w, N, crop)
    dw = oaa.conv_bwd_filter(x, dy, n, crop)
    torch.cuda.synchronize()
    return y, dx, dw


def all_elements(wl, crop, seed, chunk):
    """Every element of y, dx, dw of workload `wl` vs the oracle."""
    B, C, K, N, n = wl.B, wl.C, wl.K, wl.N, wl.n
    x, w, dy = gpu_inputs(B, C, K, N, n, crop, seed)
    y, dx, dw = run_ops(x, w, dy, N, n, crop)
    wh = w.cpu().numpy()
    ey, edx = Err(f"{wl.name} {crop} y"), Err(f"{wl.name} {crop} dx")
    dw_ref = np.zeros((K, C, n, n))
    for b0 in range(0, B, chunk):
        b1 = min(B, b0 + chunk)
        xs = x[b0:b1].cpu().numpy()
        dys = dy[b0:b1].cpu().numpy()
        ey.add(y[b0:b1].double().cpu().numpy(), oracle.conv_fwd(xs, wh, crop))
        edx.add(dx[b0:b1].double().cpu().numpy(), oracle.conv_bwd_data(dys, wh, N, crop))
        dw_ref += oracle.conv_bwd_filter(xs, dys, n, crop)
    edw = Err(f"{wl.name} {crop} dw")
    edw.add(dw.double().cpu().numpy(), dw_ref)
    return ey.check(), edx.check(), edw.check()


@pytest.mark.parametrize("crop", ["valid", "full", "same"])
def test_headline_every_element(crop):
    """BASELINE configs[1] (N=224, n=8, C=3, K=64, B=128): all 385 M elements of y, all
    19 M of dx, all 12 288 of dw, for each crop."""
    all_elements(CONFIGS["headline"], crop, seed=10, chunk=16)


def test_headline_oas_every_element():
    """NEXT-2 overlap-and-save forward at the headline size: all 385 M elements of y."""
    wl = CONFIGS["headline"]
    B, C, K, N, n, crop = wl.B, wl.C, wl.K, wl.N, wl.n, "valid"
    x, w, _ = gpu_inputs(B, C, K, N, n, crop, seed=15)
    y = oaa.conv_fwd_oas(x, w, crop)
    torch.cuda.synchronize()
    wh = w.cpu().numpy()
    e = Err("headline oas y")
    for b0 in range(0, B, 16):
        e.add(y[b0:b0 + 16].double().cpu().numpy(), oracle.conv_fwd(x[b0:b0 + 16].cpu().numpy(), wh, crop))
    e.check()


def test_alexnet_every_element():
    """BASELINE configs[3] (N=27, n=5, C=96, K=256, B=256): the tensor-core path, every
    element; dw sums a 6 400-term reduction per element (split-K + fp64 finalize)."""
    all_elements(CONFIGS["alexnet"], "valid", seed=11, chunk=32)


@pytest.mark.parametrize("wl", SWEEP, ids=lambda w: w.name)
def test_sweep_point_every_element(wl):
    """BASELINE configs[2]: the 20 (N, n) points at C=3, K=64, B=128, every element."""
    all_elements(wl, "valid", seed=12, chunk=32)


def _whole_images(x, w, dy, y, dx, imgs, N, n, crop, what):
    wh = w.cpu().numpy()
    ey, edx = Err(f"{what} y images {imgs}"), Err(f"{what} dx images {imgs}")
    for b in imgs:
        xs = x[b:b + 1].cpu().numpy()
        dys = dy[b:b + 1].cpu().numpy()
        ey.add(y[b:b + 1].double().cpu().numpy(), oracle.conv_fwd(xs, wh, crop))
        edx.add(dx[b:b + 1].double().cpu().numpy(), oracle.conv_bwd_data(dys, wh, N, crop))
    ey.check()
    edx.check()


def _dw_stratified(x, dy, dw, n, crop, what, pairs, per_pair=False):
    """Every (u, v) of the given (k, c) pairs, each a sum over the whole batch.  per_pair:
    hand the oracle only the x[:, c] and dy[:, k] planes of one pair at a time (for
    batches whose whole x and dy would not fit the host)."""
    e = Err(f"{what} dw {len(pairs)} (k,c) pairs")
    uv = [(u, v) for u in range(n) for v in range(n)]
    if per_pair:
        for (k, c) in pairs:
            idx = np.array([(0, 0, u, v) for (u, v) in uv], dtype=np.int64)
            ref = oracle.bwd_filter_sample(x[:, c:c + 1].contiguous().cpu().numpy(),
                                           dy[:, k:k + 1].contiguous().cpu().numpy(), n, crop, idx)
            e.add(dw[k, c].reshape(-1).double().cpu().numpy(), ref)
    else:
        idx = np.array([(k, c, u, v) for (k, c) in pairs for (u, v) in uv], dtype=np.int64)
        ref = oracle.bwd_filter_sample(x.cpu().numpy(), dy.cpu().numpy(), n, crop, idx)
        got = dw[tuple(torch.from_numpy(idx[:, i]).cuda() for i in range(4))].double().cpu().numpy()
        e.add(got, ref)
    # the whole-tensor scale: rel-L2 of the sampled pairs against their own norm, max
    # against the largest sampled reference (a lower bound of max|dw|)
    e.check()


def _adjoint(y, dy, x, dx, w, dw):
    """⟨fwd(x,w), dy⟩ = ⟨x, bwd_data(dy,w)⟩ = ⟨w, bwd_filter(x,dy)⟩ (the exact adjoint
    identity of the three definitions, SURVEY.md §8(c) pins)."""
    a = float((y.double() * dy.double()).sum())
    b = float((x.double() * dx.double()).sum())
    c = float((w.double() * dw.double()).sum())
    scale = math.sqrt(float((y.double() ** 2).sum()) * float((dy.double() ** 2).sum()))
    assert abs(a - b) <= 1e-6 * scale, (a, b, scale)
    assert abs(a - c) <= 1e-6 * scale, (a, c, scale)


def test_sharded_shard_full_size():
    """configs[4]'s per-GPU shard at G = 8 (B = 128 of 1024, C=64, K=128): whole images
    0, 77 and 127 (every element of y and dx), dw at one (k, c) pair per output channel k
    (all 128 rows of the bin GEMM's M tile, c striding over all 64 input channels) and
    per input channel c, plus the adjoint identity over the full tensors."""
    c5 = CONFIGS["sharded"]
    B, C, K, N, n, crop = 128, c5.C, c5.K, c5.N, c5.n, "valid"
    x, w, dy = gpu_inputs(B, C, K, N, n, crop, seed=13)
    y, dx, dw = run_ops(x, w, dy, N, n, crop)
    _whole_images(x, w, dy, y, dx, [0, 77, 127], N, n, crop, "sharded shard")
    pairs = sorted({(k, (7 * k + 3) % C) for k in range(K)} | {((5 * c + 1) % K, c) for c in range(C)})
    _dw_stratified(x, dy, dw, n, crop, "sharded shard", pairs)
    _adjoint(y, dy, x, dx, w, dw)


def test_alexnet_fused_backward_every_element():
    """NEXT-1 fused backward at configs[3] (tensor-core path, dy spectra shared by both
    GEMMs): every element of dx and dw."""
    wl = CONFIGS["alexnet"]
    B, C, K, N, n, crop = wl.B, wl.C, wl.K, wl.N, wl.n, "valid"
    x, w, dy = gpu_inputs(B, C, K, N, n, crop, seed=16)
    dx, dw = oaa.conv_bwd(x, dy, w, crop)
    torch.cuda.synchronize()
    wh = w.cpu().numpy()
    edx, edw = Err("alexnet fused dx"), Err("alexnet fused dw")
    dw_ref = np.zeros((K, C, n, n))
    for b0 in range(0, B, 32):
        xs, dys = x[b0:b0 + 32].cpu().numpy(), dy[b0:b0 + 32].cpu().numpy()
        edx.add(dx[b0:b0 + 32].double().cpu().numpy(), oracle.conv_bwd_data(dys, wh, N, crop))
        dw_ref += oracle.conv_bwd_filter(xs, dys, n, crop)
    edw.add(dw.double().cpu().numpy(), dw_ref)
    edx.check()
    edw.check()


def test_config5_global_batch_one_gpu():
    """configs[4] at its global batch B = 1024 on one GPU (N=1 of the strong-scaling run):
    whole images 0, 511 and 1023; dw against the fp64 sum of the eight B = 128 shard calls
    the 8-GPU run makes (the all-reduce of SURVEY.md §8(e), done here on one device), and
    against the oracle at stratified (k, c) pairs over the whole 1024-image batch."""
    c5 = CONFIGS["sharded"]
    B, C, K, N, n, crop = c5.B, c5.C, c5.K, c5.N, c5.n, "valid"
    x, w, dy = gpu_inputs(B, C, K, N, n, crop, seed=14)
    y, dx, dw = run_ops(x, w, dy, N, n, crop)
    _whole_images(x, w, dy, y, dx, [0, 511, 1023], N, n, crop, "config5 B=1024")
    del dx
    shards = torch.zeros((K, C, n, n), dtype=torch.float64, device="cuda")
    for r in range(8):
        shards += oaa.conv_bwd_filter(x[128 * r:128 * (r + 1)], dy[128 * r:128 * (r + 1)], n, crop).double()
    e = Err("config5 dw vs Σ of 8 shard dw")
    e.add(dw.double().cpu().numpy(), shards.cpu().numpy())
    e.check()
    pairs = [(k, (11 * k + 5) % C) for k in range(0, K, 8)]
    _dw_stratified(x, dy, dw, n, crop, "config5 B=1024", pairs, per_pair=True)
    del y
    torch.cuda.empty_cache()
