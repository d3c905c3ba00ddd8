"""Roofline model of the OaA layer, shared by bench.py and tools/sweep.py.

Algorithmic work per pass (what OaA must move or compute, not the dense work it avoids):
  bytes : 4·(B·C·N² + K·C·n² + B·K·M²)  -- each pass reads two of x / w / dy and writes the
          third; spectra are on-chip intermediates and are not counted
  alu   : 5·P²·log2(P) flops per real P×P transform (the FFT convention; half of
          5·L·log2(L) for L = P²), B·(C+K)·T of them plus the K·C weight transforms,
          + P² adds per output block for the overlap-add
  tc    : 8·K·C·B·T·bins, the per-bin complex channel contraction (a4)
with T = ceil(N/n)² blocks for the forward, T' = ceil(M/n)² dy blocks for the backward.

T_roof = max(T_HBM, T_ALU, T_TC) with the denominators
  HBM  MEASURED_PEAKS.json hbm_gbs (driver-measured copy bandwidth),
  ALU  fp32 FFMA measured by tools/microbench/peaks.cu (profiles/peaks_r02.json),
  TC   fp32-accurate 3×TF32 = the measured tcgen05 kind::tf32 peak / 3,
each with a documented fallback when the file is absent.

Per-kernel attribution: each kernel of the library is charged the part of its op's
algorithmic work that it performs (KERNEL_WORK below), so the dominant kernel's roofline
fraction is T_roof(kernel) / t(kernel).
"""
from __future__ import annotations

import json
import math
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def out_size(N, n, crop):
    return {"full": N + n - 1, "valid": N - n + 1, "same": N}[crop]


def peaks():
    """(hbm GB/s, ffma TFLOP/s, 3×TF32 TFLOP/s, source notes)."""
    src = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            hbm = float(json.load(f)["hbm_gbs"])
        src["hbm"] = "MEASURED_PEAKS.json hbm_gbs (driver-measured)"
    except Exception:
        hbm = 6650.0
        src["hbm"] = "fallback 6650 GB/s (B200_PROFILING.md)"
    try:
        with open(os.path.join(ROOT, "profiles", "peaks_r02.json")) as f:
            pk = json.load(f)
        ffma = float(pk["ffma_tflops"])
        tc3 = float(pk["tcgen05_tf32_tflops"]) / 3.0
        src["alu"] = "fp32 FFMA measured on B200 (tools/microbench/peaks.cu, profiles/peaks_r02.json)"
        src["tc"] = "tcgen05 kind::tf32 measured on B200 / 3 for 3xTF32 (profiles/peaks_r02.json)"
    except Exception:
        ffma = 2 * 148 * 128 * 1.965e9 / 1e12
        tc3 = 1100.0 / 3.0
        src["alu"] = "derived 148 SM x 128 lanes x 2 x 1965 MHz"
        src["tc"] = "nominal dense TF32 1100 TFLOP/s / 3"
    return hbm, ffma, tc3, src


def geometry(B, C, K, N, n, crop):
    M = out_size(N, n, crop)
    P = 2 * n - 1
    return dict(M=M, P=P, bins=P * n, T=math.ceil(N / n) ** 2, Td=math.ceil(M / n) ** 2,
                fft=5 * P * P * math.log2(P) if P > 1 else 1.0)


def op_work(op, B, C, K, N, n, crop):
    """{'bytes', 'alu', 'tc'} of one pass."""
    g = geometry(B, C, K, N, n, crop)
    by = 4 * (B * C * N * N + K * C * n * n + B * K * g["M"] ** 2)
    wt = K * C * g["fft"]
    if op == "fwd":
        T = g["T"]
        alu = B * (C + K) * T * g["fft"] + g["P"] ** 2 * B * K * T + wt
    elif op == "bwd_data":
        T = g["Td"]
        alu = B * (C + K) * T * g["fft"] + g["P"] ** 2 * B * C * T + wt
    elif op == "bwd_filter":
        T = g["Td"]
        alu = B * (C + K) * T * g["fft"] + wt
    else:
        raise ValueError(op)
    return {"bytes": by, "alu": alu, "tc": 8 * K * C * B * T * g["bins"]}


def kernel_work(kname, op, B, C, K, N, n, crop):
    """The part of op `op`'s algorithmic work that kernel `kname` performs."""
    g = geometry(B, C, K, N, n, crop)
    M, P, fft = g["M"], g["P"], g["fft"]
    T = g["T"] if op == "fwd" else g["Td"]
    cin, cout = (C, K) if op == "fwd" else (K, C)
    rin, rout = (N, M) if op == "fwd" else (M, N)
    z = {"bytes": 0.0, "alu": 0.0, "tc": 0.0}
    if kname in ("spectrum", "finalize"):
        return {**z, "bytes": 4 * K * C * n * n, "alu": K * C * fft}
    if kname in ("xspec", "tile_spectra") and op != "bwd_filter":
        return {**z, "bytes": 4 * B * cin * rin * rin, "alu": B * cin * T * fft}
    if kname in ("walk", "walk_load"):
        return {**z, "bytes": 4 * B * cout * rout * rout, "alu": B * cout * T * (fft + P * P),
                "tc": 8 * K * C * B * T * g["bins"] if kname == "walk" else 0.0}
    if kname == "bin_gemm":
        return {**z, "tc": 8 * K * C * B * T * g["bins"]}
    if kname == "bwdd":
        return op_work("bwd_data", B, C, K, N, n, crop) | {"alu": B * (C + K) * T * fft + P * P * B * C * T}
    if kname == "xspec_win":
        return {**z, "bytes": 4 * B * C * N * N, "alu": B * C * T * fft}
    if kname == "bwdf":
        return {**z, "bytes": 4 * B * K * M * M, "alu": B * K * T * fft, "tc": 8 * K * C * B * T * g["bins"]}
    if kname == "filter_spectra":
        return {**z, "bytes": 4 * (B * K * M * M + B * C * N * N), "alu": B * (C + K) * T * fft}
    if kname == "engine":
        return op_work(op, B, C, K, N, n, crop)
    return z


def t_roof(work):
    """(T_roof seconds, bound, per-term seconds) for a work dict."""
    hbm, ffma, tc3, _ = peaks()
    terms = {"hbm": work["bytes"] / (hbm * 1e9), "alu": work["alu"] / (ffma * 1e12),
             "tc": work["tc"] / (tc3 * 1e12)}
    bound = max(terms, key=terms.get)
    return terms[bound], bound, terms


def roofline_record(work, seconds):
    """The bench.py `roofline` object for a kernel doing `work` in `seconds` per launch."""
    hbm, ffma, tc3, src = peaks()
    T, bound, terms = t_roof(work)
    if bound == "hbm":
        achieved, peak, unit, q = work["bytes"] / seconds / 1e9, hbm, "GB/s", "bytes"
    elif bound == "alu":
        achieved, peak, unit, q = work["alu"] / seconds / 1e12, ffma, "TFLOP/s", "alu"
    else:
        achieved, peak, unit, q = work["tc"] / seconds / 1e12, tc3, "TFLOP/s", "tc"
    return {"bound": {"hbm": "hbm", "alu": "alu", "tc": "tensor"}[bound], "achieved": achieved, "peak": peak,
            "unit": unit, "frac": achieved / peak, "t_roof_ms": T * 1e3, "kernel_ms": seconds * 1e3,
            "terms_ms": {k: v * 1e3 for k, v in terms.items()}, "peak_source": src[bound],
            "algorithmic": {"bytes": work["bytes"], "alu_flops": work["alu"], "tc_flops": work["tc"]}}


def direct_flops(B, C, K, N, n, crop, passes=3):
    """Direct-convolution flops (TFLOP-equivalent convention): passes × 2·B·K·C·n²·M²."""
    M = out_size(N, n, crop)
    return passes * 2 * B * K * C * n * n * M * M
