"""CPU-side checks of the C-ABI library (no GPU needed, no compute launched):
liboaa.so builds/loads, exports every symbol include/oaa.h declares, and its host-side
argument validation / size bookkeeping behave as documented.  Validation runs before
any CUDA call, so invalid arguments can be exercised without a device."""
import ctypes
import os
import re

import pytest

import paper_1601_06815_b200 as oaa
from workloads import out_size as ref_out_size

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "oaa.h")).read()
    return sorted(set(re.findall(r"\b(oaa_[a-z_]+)\s*\(", hdr)))


def test_header_symbols_exported():
    L = oaa.lib()
    syms = declared_symbols()
    assert {"oaa_conv_fwd", "oaa_conv_bwd_data", "oaa_conv_bwd_filter"} <= set(syms)
    for s in syms:
        assert hasattr(L, s), f"liboaa.so does not export {s}"


def test_version():
    assert "sm_100a" in oaa.version()


@pytest.mark.parametrize("crop", ["full", "valid", "same"])
@pytest.mark.parametrize("N,n", [(1, 1), (5, 3), (32, 3), (224, 8), (27, 5), (3, 5), (8, 8)])
def test_out_size_matches_convmode(N, n, crop):
    if crop == "valid" and n > N:
        with pytest.raises(ValueError):
            oaa.out_size(N, n, crop)
        return
    assert oaa.out_size(N, n, crop) == ref_out_size(N, n, crop)


def _call(name, B=1, C=1, K=1, N=8, n=3, crop=1, ptrs=(0x1000, 0x200000, 0x40000000),
          ws=0x7000000000, ws_bytes=1 << 30):
    f = getattr(oaa.lib(), name)
    return f(ctypes.c_void_p(ptrs[0]), ctypes.c_void_p(ptrs[1]), ctypes.c_void_p(ptrs[2]),
             B, C, K, N, n, crop, ctypes.c_void_p(ws), ctypes.c_size_t(ws_bytes), None)


@pytest.mark.parametrize("name", ["oaa_conv_fwd", "oaa_conv_bwd_data", "oaa_conv_bwd_filter", "oaa_conv_fwd_oas",
                                  "oaa_conv_fwd_prepared", "oaa_conv_bwd_data_prepared"])
def test_invalid_arguments_rejected_before_launch(name):
    INVALID, UNSUP = 1, 2
    assert _call(name, B=-1) == INVALID
    assert _call(name, C=0) == INVALID
    assert _call(name, K=0) == INVALID
    assert _call(name, N=0) == INVALID
    assert _call(name, n=0) == INVALID
    assert _call(name, crop=7) == INVALID
    assert _call(name, N=3, n=5, crop=1) == INVALID          # Valid needs n <= N
    assert _call(name, ptrs=(0, 0x200000, 0x40000000)) == INVALID
    assert _call(name, n=9, N=20) == UNSUP                      # v1: n <= 8
    assert _call(name, N=2000, n=3) == UNSUP                    # max(ceil(N/n)·n, M) ≤ 256


def test_aliasing_rejected():
    # output range overlapping an input range
    assert _call("oaa_conv_fwd", ptrs=(0x1000, 0x200000, 0x1000)) == 1


def test_workspace_sizes():
    for op in (oaa.OP_FWD, oaa.OP_BWD_DATA, oaa.OP_BWD_FILTER):
        assert oaa.workspace_bytes(op, 128, 3, 64, 224, 8, "valid") > 0
        assert oaa.workspace_bytes(op, 128, 3, 64, 224, 8, "valid") % 256 == 0
        assert oaa.workspace_bytes(op, 0, 3, 64, 224, 8, "valid") == 0
        assert oaa.workspace_bytes(op, 1, 3, 64, 3, 5, "valid") == 0    # invalid -> 0
    # too-small workspace is reported, not overrun
    assert _call("oaa_conv_fwd", N=32, n=3, ws_bytes=16) == 3


def test_status_strings():
    L = oaa.lib()
    for s in range(5):
        assert L.oaa_status_string(s)


def test_missing_extension_fails_loudly(monkeypatch):
    import paper_1601_06815_b200 as pkg
    monkeypatch.setattr(pkg, "_lib", None)
    monkeypatch.setattr(pkg, "_LIB_PATH", "/nonexistent/liboaa.so")
    with pytest.raises(pkg.OaAError):
        pkg.lib()


def test_cpu_tensors_rejected():
    import torch
    x = torch.zeros(1, 1, 8, 8)
    w = torch.zeros(1, 1, 3, 3)
    with pytest.raises(ValueError):
        oaa.conv_fwd(x, w)


def _bwd(B=1, C=1, K=1, N=8, n=3, crop=1, ptrs=(0x1000, 0x200000, 0x40000000, 0x80000000, 0xC0000000),
         ws=0x7000000000, ws_bytes=1 << 30):
    P = ctypes.c_void_p
    return oaa.lib().oaa_conv_bwd(*(P(p) for p in ptrs), B, C, K, N, n, crop, P(ws), ctypes.c_size_t(ws_bytes), None)


def test_fused_backward_validation():
    """oaa_conv_bwd (NEXT-1) validates like the two separate calls, plus pairwise
    disjointness of x, dy, w, dx, dw."""
    INVALID, UNSUP, WS = 1, 2, 3
    assert _bwd(B=-1) == INVALID
    assert _bwd(C=0) == INVALID
    assert _bwd(N=3, n=5) == INVALID
    assert _bwd(n=9, N=20) == UNSUP
    assert _bwd(ptrs=(0x1000, 0x200000, 0, 0x80000000, 0xC0000000)) == INVALID       # null w
    assert _bwd(ptrs=(0x1000, 0x200000, 0x40000000, 0x1000, 0xC0000000)) == INVALID  # dx aliases x
    assert _bwd(ptrs=(0x1000, 0x200000, 0x40000000, 0x80000000, 0x40000000)) == INVALID  # dw aliases w
    assert _bwd(N=32, n=8, ws_bytes=16) == WS


def test_new_op_workspace_sizes():
    for op in (oaa.OP_FWD_OAS, oaa.OP_BWD):
        assert oaa.workspace_bytes(op, 128, 3, 64, 224, 8, "valid") > 0
        assert oaa.workspace_bytes(op, 128, 3, 64, 224, 8, "valid") % 256 == 0
    # the fused backward needs at least what the two separate ops need on the SIMT path
    assert oaa.workspace_bytes(oaa.OP_BWD, 256, 96, 256, 27, 5, "valid") > 0
    assert oaa.workspace_bytes(oaa.OP_FWD_OAS, 2, 5, 3, 16, 3, "valid") == 0   # OaS: C ≤ 4 or C, K ≥ 16
    # OaS on the tensor-core path (C, K ≥ 16): the engine layout over the ⌈M/n⌉² output tiles
    tc = oaa.workspace_bytes(oaa.OP_FWD_OAS, 4, 32, 32, 32, 8, "valid")
    assert tc > 0 and tc % 256 == 0
    assert oaa.workspace_bytes(oaa.OP_FWD_OAS, 4, 32, 32, 32, 8, "full") >= tc  # more output tiles
    L = oaa.lib()
    for op in (oaa.OP_FWD, oaa.OP_BWD_DATA):
        assert L.oaa_weight_spectra_bytes(op, 3, 64, 224, 8, 1) % 256 == 0
        assert L.oaa_weight_spectra_bytes(op, 3, 64, 224, 8, 1) >= 16 * 3 * 64 * 64
    assert L.oaa_weight_spectra_bytes(oaa.OP_BWD_FILTER, 3, 64, 224, 8, 1) == 0
    # too-small spectra buffer / bad op are reported before any launch
    P = ctypes.c_void_p
    assert L.oaa_weight_spectra(oaa.OP_FWD, P(0x1000), P(0x7000000000), 16, 3, 64, 224, 8, 1, None) == 3
    assert L.oaa_weight_spectra(oaa.OP_BWD_FILTER, P(0x1000), P(0x7000000000), 1 << 20, 3, 64, 224, 8, 1, None) == 1


def test_block_size_planning():
    """DESIGN.md R18 (SURVEY.md §8(f) NEXT-4 "block size b != n"): the forward walker and bwd_data
    (C <= 4 output channels) tile into b = 16 - n blocks (P = 15) for 3 <= n <= 7 once the image
    holds >= 3 of them (bwd_data: n <= 4, or >= 96 pixels per side); everything else keeps the
    paper's b = n.  Host planning only -- no GPU needed."""
    bs = oaa.block_size
    # the BASELINE sweep at N = 224 and 128 (C = 3, K = 64): larger blocks in both ops
    for N in (224, 128):
        for n in (3, 5, 7):
            assert bs("fwd", 3, 64, N, n) == 16 - n
            assert bs("bwd_data", 3, 64, N, n) == 16 - n
        assert bs("fwd", 3, 64, N, 8) == 8 and bs("bwd_data", 3, 64, N, 8) == 8
    # thresholds: fwd from N >= 3b, or from 2b with <= 1.5x the area in padded blocks; bwd_data
    # (dy side M) from 3b for n <= 4, from 96 for n >= 5
    assert bs("fwd", 1, 1, 39, 3) == 13 and bs("fwd", 1, 1, 38, 3) == 13 and bs("fwd", 1, 1, 32, 3) == 13
    assert bs("fwd", 1, 1, 27, 3) == 3 and bs("fwd", 1, 1, 25, 3) == 3     # 39²/27² > 1.5; < 2b
    assert bs("fwd", 1, 1, 27, 7, "same") == 9 and bs("fwd", 1, 1, 20, 7, "same") == 7
    assert bs("fwd", 3, 64, 32, 5) == 11 and bs("fwd", 3, 64, 16, 5) == 5
    assert bs("bwd_data", 3, 8, 64, 5) == 5          # M = 60 < 96
    assert bs("bwd_data", 3, 8, 64, 3) == 13         # M = 62 >= 39
    # n = 1, 2 and the tensor-core path (C, K >= 16) keep b = n; so does any op with C > 4 inputs
    assert bs("fwd", 3, 8, 224, 2) == 2 and bs("fwd", 3, 8, 224, 1) == 1
    assert bs("fwd", 64, 128, 224, 5) == 5 and bs("bwd_data", 64, 128, 224, 5) == 5
    assert bs("fwd", 96, 256, 27, 5) == 5                       # configs[3]: b = n
    assert bs("fwd", 32, 64, 64, 7) == 9 and bs("bwd_data", 32, 64, 64, 7) == 9  # TC path, prime P = 13
    assert bs("fwd", 6, 7, 224, 3) == 3
    assert oaa.lib().oaa_block_size(2, 3, 64, 224, 3, 1) == -1  # bwd_filter: not a block-size op
    assert oaa.lib().oaa_block_size(0, 3, 64, 2, 3, 1) == -1    # Valid with n > N
    with pytest.raises(ValueError):
        bs("bwd_filter", 3, 64, 224, 3)
