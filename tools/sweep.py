"""Time every BASELINE.json config (headline, the N × n sweep, AlexNet-like, the per-GPU
shard of the sharded config) pass by pass with CUDA events and report, per config, the
step time, images/s, TFLOP-equivalent/s (direct-convolution flops) and the
fractions of the ALU (FFT-convention flops) and HBM (algorithmic bytes) rooflines.

    python tools/sweep.py [--out profiles/r1_sweep.md] [--reps 5]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1601_06815_b200 as oaa  # noqa: E402
from tools import roofline as rl  # noqa: E402
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
    # the whole step captured once into a CUDA graph and replayed (removes the host launch
    # latency of the ~8 launches per step, which dominates the small-N points)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for f in ops.values():
            f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for f in ops.values():
            f()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); g.replay(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    ts.sort()
    res["graph_step"] = ts[len(ts) // 2]
    del g
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
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_sweep.md"))
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    hbm, ffma, tc3, src = rl.peaks()
    wls = [CONFIGS["headline"]] + list(SWEEP) + [CONFIGS["alexnet"]]
    sh = CONFIGS["sharded"]
    from workloads import Workload
    wls.append(Workload("sharded_per_gpu_B128", B=128, C=sh.C, K=sh.K, N=sh.N, n=sh.n))
    if args.only:
        wls = [w for w in wls if args.only in w.name]
    rows = []
    for wl in wls:
        t = time_config(wl, args.reps)
        graph_step = t.pop("graph_step")
        step = sum(t.values())
        dims = (wl.B, wl.C, wl.K, wl.N, wl.n, wl.crop)
        roof = {op: rl.t_roof(rl.op_work(op, *dims)) for op in t}
        t_roof = sum(r[0] for r in roof.values())
        bounds = sorted(set(r[1] for r in roof.values()))
        r = dict(config=wl.name, B=wl.B, C=wl.C, K=wl.K, N=wl.N, n=wl.n,
                 ms={k: round(v, 4) for k, v in t.items()}, step_ms=round(step, 4),
                 images_per_s=wl.B / (step / 1e3), tflop_eq_per_s=rl.direct_flops(*dims) / (step / 1e3) / 1e12,
                 roofline_bound="/".join(bounds), roofline_frac=t_roof * 1e3 / step,
                 graph_step_ms=round(graph_step, 4), graph_frac=t_roof * 1e3 / graph_step,
                 op_frac={op: roof[op][0] * 1e3 / t[op] for op in t})
        rows.append(r)
        print(json.dumps(r), flush=True)
    lines = ["# Sweep: every BASELINE.json config on one B200 (tools/sweep.py)", "",
             f"CUDA events, median of {args.reps} per pass (passes timed one after another), inputs "
             "device-resident, Valid crop. Roofline (SURVEY.md §8(d), tools/roofline.py): per pass "
             "T_roof = max(T_HBM, T_ALU of the FFTs + overlap-add, T_TC of the contraction); "
             f"denominators HBM {hbm:.0f} GB/s ({src['hbm']}), FFMA {ffma:.1f} TFLOP/s ({src['alu']}), "
             f"3xTF32 {tc3:.0f} TFLOP/s ({src['tc']}). frac = Σ_pass T_roof / step time. "
             "TFLOP-eq/s counts the direct-convolution flops (3 passes × 2·B·K·C·n²·M²). 'graph step': the "
             "three passes captured once into a CUDA graph and replayed (no host launch latency).", "",
             "| config | B | C | K | N | n | fwd ms | bwd_data ms | bwd_filter ms | step ms | images/s | TFLOP-eq/s | bound | step frac | fwd / bwd_d / bwd_f frac | graph step ms | graph frac |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        of = r["op_frac"]
        lines.append(f"| {r['config']} | {r['B']} | {r['C']} | {r['K']} | {r['N']} | {r['n']} | {r['ms']['fwd']:.3f} | "
                     f"{r['ms']['bwd_data']:.3f} | {r['ms']['bwd_filter']:.3f} | {r['step_ms']:.3f} | "
                     f"{r['images_per_s']:.0f} | {r['tflop_eq_per_s']:.1f} | {r['roofline_bound']} | "
                     f"{r['roofline_frac']:.2f} | {of['fwd']:.2f} / {of['bwd_data']:.2f} / {of['bwd_filter']:.2f} | "
                     f"{r['graph_step_ms']:.3f} | {r['graph_frac']:.2f} |")
    with open(args.out, "w") as f:
        f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
