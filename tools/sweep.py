"""Time every BASELINE.json config (headline, the N × n sweep, AlexNet-like, the per-GPU
shard of the sharded config) pass by pass with CUDA events and report, per config, the
step time, images/s, TFLOP-equivalent/s (direct-convolution flops) and the
fractions of the ALU (FFT-convention flops) and HBM (algorithmic bytes) rooflines.

    python tools/sweep.py [--out profiles/r1_sweep.md] [--reps 5]
"""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1601_06815_b200 as oaa  # noqa: E402
from bench import algorithmic_terms, measured_peaks  # noqa: E402
from workloads import CONFIGS, SWEEP, out_size  # noqa: E402


def time_config(wl, reps):
    B, C, K, N, n, crop = wl.B, wl.C, wl.K, wl.N, wl.n, wl.crop
    M = out_size(N, n, crop)
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.rand((B, C, N, N), generator=g, device="cuda") * 2 - 1
    w = torch.rand((K, C, n, n), generator=g, device="cuda") * 2 - 1
    dy = torch.rand((B, K, M, M), generator=g, device="cuda") * 2 - 1
    y = torch.empty((B, K, M, M), device="cuda"); dx = torch.empty_like(x); dw = torch.empty_like(w)
    ops = {"fwd": lambda: oaa.conv_fwd(x, w, crop, out=y),
           "bwd_data": lambda: oaa.conv_bwd_data(dy, w, N, crop, out=dx),
           "bwd_filter": lambda: oaa.conv_bwd_filter(x, dy, n, crop, out=dw)}
    res = {}
    for name, f in ops.items():
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(); f(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
        ts.sort()
        res[name] = ts[len(ts) // 2]
    del x, w, dy, y, dx, dw
    torch.cuda.empty_cache()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r1_sweep.md"))
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    peaks, src = measured_peaks()
    sm_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    alu_peak = 2 * 148 * 128 * sm_mhz * 1e6  # flop/s
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0)) * 1e9
    # fp32-accurate tensor rate: TF32 dense = bf16 × (1.1 / 2.25) (B200_PROFILING.md nominal ratio), / 3 for 3×TF32
    tc_peak = float(peaks.get("bf16_tflops", 1590.0)) * 1e12 * (1.1 / 2.25) / 3
    wls = [CONFIGS["headline"]] + list(SWEEP) + [CONFIGS["alexnet"]]
    sh = CONFIGS["sharded"]
    from workloads import Workload
    wls.append(Workload("sharded_per_gpu_B128", B=128, C=sh.C, K=sh.K, N=sh.N, n=sh.n))
    rows = []
    for wl in wls:
        t = time_config(wl, args.reps)
        d = dict(name=wl.name, B=wl.B, C=wl.C, K=wl.K, N=wl.N, n=wl.n, crop=wl.crop)
        terms = algorithmic_terms(d)
        step = sum(t.values())
        M = out_size(wl.N, wl.n, wl.crop)
        direct = 3 * 2 * wl.B * wl.K * wl.C * wl.n ** 2 * M ** 2
        t_alu = sum(terms["flops"].values()) / alu_peak
        t_hbm = sum(terms["bytes"].values()) / hbm_peak
        # SURVEY.md §8(d) roofline: T_roof = max(T_HBM, T_ALU(FFTs + overlap-add), T_TC(contraction
        # at the fp32-accurate 3×TF32 rate)); the tensor-core path is taken for C, K ≥ 16
        P = 2 * wl.n - 1
        bins = P * wl.n
        T = math.ceil(wl.N / wl.n) ** 2
        Td = math.ceil(M / wl.n) ** 2
        contraction = 8 * wl.K * wl.C * wl.B * bins * (T + 2 * Td)
        t_fft = (sum(terms["flops"].values()) - contraction) / alu_peak
        t_tc = contraction / tc_peak
        t_roof = max(t_hbm, t_fft, t_tc)
        bound = {t_hbm: "HBM", t_fft: "ALU", t_tc: "TC"}[t_roof]
        r = dict(config=wl.name, B=wl.B, C=wl.C, K=wl.K, N=wl.N, n=wl.n,
                 ms={k: round(v, 4) for k, v in t.items()}, step_ms=round(step, 4),
                 images_per_s=wl.B / (step / 1e3), tflop_eq_per_s=direct / (step / 1e3) / 1e12,
                 alu_roofline_frac=t_alu / (step / 1e3), hbm_roofline_frac=t_hbm / (step / 1e3),
                 roofline_bound=bound, roofline_frac=t_roof / (step / 1e3))
        rows.append(r)
        print(json.dumps(r), flush=True)
    lines = ["# r1 sweep: every BASELINE.json config on one B200 (tools/sweep.py)", "",
             f"CUDA events, median of {args.reps} per pass, inputs device-resident, Valid crop. "
             f"Roofline denominators: fp32 FFMA {alu_peak / 1e12:.1f} TFLOP/s (148 SM × 128 lanes × 2 × "
             f"{sm_mhz:.0f} MHz) for the FFT-convention flops of SURVEY.md §8(d), HBM {hbm_peak / 1e9:.0f} GB/s "
             f"({src}) for the algorithmic bytes. TFLOP-eq/s counts the direct-convolution flops "
             "(3 passes × 2·B·K·C·n²·M²), the convention for FFT-convolution layers. "
             f"Roofline (SURVEY.md §8(d)): T_roof = max(T_HBM, T_ALU of the FFTs + overlap-add, T_TC of the "
             f"contraction at the fp32-accurate 3×TF32 rate {tc_peak / 1e12:.0f} TFLOP/s = bf16 peak × 1.1/2.25 / 3); "
             "'ALU frac (FMA path)' also counts the contraction on the FMA pipe, as the small-C kernels do.", "",
             "| config | B | C | K | N | n | fwd ms | bwd_data ms | bwd_filter ms | step ms | images/s | TFLOP-eq/s | bound | roofline frac | ALU frac (FMA path) | HBM frac |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        lines.append(f"| {r['config']} | {r['B']} | {r['C']} | {r['K']} | {r['N']} | {r['n']} | {r['ms']['fwd']:.3f} | "
                     f"{r['ms']['bwd_data']:.3f} | {r['ms']['bwd_filter']:.3f} | {r['step_ms']:.3f} | "
                     f"{r['images_per_s']:.0f} | {r['tflop_eq_per_s']:.1f} | {r['roofline_bound']} | "
                     f"{r['roofline_frac']:.2f} | {r['alu_roofline_frac']:.2f} | {r['hbm_roofline_frac']:.2f} |")
    with open(args.out, "w") as f:
        f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
