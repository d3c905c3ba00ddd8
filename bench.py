#!/usr/bin/env python
"""Benchmark of the OaA convolution layer (arXiv 1601.06815) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...        (N > 1)

A step is one pass of the whole hot path -- forward, bwd_data, bwd_filter (PAPER.md:89
"two actual convolutions per kernel" in the backward) -- over one batch of the headline
workload (BASELINE.json configs[1]: N=224, n=8, C=3, K=64, B=128 per GPU, Valid crop),
plus the NCCL all-reduce of dW when N > 1 (batch sharding, weak scaling: every GPU
processes B=128 images).  Prints ONE JSON line (rank 0).

  value     images/s of the whole job, device-resident inputs, CUDA-event timed region
            (barrier + synchronize on both sides, max over ranks).
  e2e       the same metric through the public API with PINNED HOST buffers: the
            host→device copies of x, w, dy and the device→host copies of y, dx, dw are
            inside the timed region.
  roofline  the dominant kernel's algorithmic FLOPs per launch (SURVEY.md §8(d)
            convention) ÷ its CUDA-event duration inside the timed
            region, against the fp32 FFMA peak derived in DESIGN.md.
  cpu_baseline  the CPU float64 oracle (direct definition) on the host cores, on a
            bounded sample of the same workload.
--impl reference runs that oracle as the reference arm (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HEAD = dict(name="headline", B=128, C=3, K=64, N=224, n=8, crop="valid")
METRIC = "OaA conv fwd+bwd images/s at N=224,n=8,C=3,K=64; % of HBM/tensor roofline"
UNIT = "images/s"
SM_COUNT = 148
FP32_LANES_PER_SM = 128


def workload_name(w):
    return f"headline N={w['N']} n={w['n']} C={w['C']} K={w['K']} B={w['B']}/gpu crop={w['crop']}"


def out_size(N, n, crop):
    return {"full": N + n - 1, "valid": N - n + 1, "same": N}[crop]


# ------------------------------------------------------------------ roofline terms
def algorithmic_terms(w):
    """Per-pass algorithmic work, for one GPU's batch.

    bytes  : 4·(B·C·N² + K·C·n² + B·K·M²)  (each pass reads two of x / w / dy and writes
             the third; spectra are on-chip intermediates, not counted)
    flops  : FFT convention 5·P²·log2(P) per real P×P transform, B·(Cin+Cout)·T of them,
             + contraction 8·Cin·Cout·bins per block, + P² overlap-add adds per output
             block (T = blocks per channel of the transformed side).
    """
    B, C, K, N, n, crop = w["B"], w["C"], w["K"], w["N"], w["n"], w["crop"]
    M = out_size(N, n, crop)
    P = 2 * n - 1
    bins = P * n
    T = math.ceil(N / n) ** 2
    Td = math.ceil(M / n) ** 2
    fft = 5 * P * P * math.log2(P) if P > 1 else 1
    by = 4 * (B * C * N * N + K * C * n * n + B * K * M * M)
    fwd = B * (C + K) * T * fft + 8 * K * C * B * T * bins + P * P * B * K * T
    bwd_data = B * (C + K) * Td * fft + 8 * K * C * B * Td * bins + P * P * B * C * Td
    bwd_filter = B * (C + K) * Td * fft + 8 * K * C * B * Td * bins
    return {"bytes": {"fwd": by, "bwd_data": by, "bwd_filter": by},
            "flops": {"fwd": fwd, "bwd_data": bwd_data, "bwd_filter": bwd_filter}}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


# ------------------------------------------------------------------ clocks sampler
class ClockSampler:
    def __init__(self, index=0, period_ms=50):
        self.index, self.period_ms = index, period_ms
        self.proc = None
        self.lines = []

    def __enter__(self):
        cmd = ["nvidia-smi", f"--id={self.index}",
               "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
               "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
               "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
               "--format=csv,noheader,nounits", f"-lms={self.period_ms}"]
        try:
            self.proc = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() in ("active", "1", "yes"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ CPU oracle timing
def cpu_oracle_rate(w, budget_s=15.0, max_images=512):
    """Time the float64 direct oracle (fwd + bwd_data + bwd_filter) on a sub-batch of
    the workload on all host cores; returns (images/s, cores, sample description)."""
    import numpy as np

    import oracle
    from workloads import make_inputs
    cores = oracle.max_threads()
    d = make_inputs(1, w["C"], w["K"], w["N"], w["n"], w["crop"], seed=7)
    t0 = time.perf_counter()
    oracle.step_f32(d["x"], d["w"], d["dy"], w["crop"])
    t1 = time.perf_counter() - t0
    nb = int(max(1, min(max_images, budget_s / max(t1, 1e-3))))
    d = make_inputs(nb, w["C"], w["K"], w["N"], w["n"], w["crop"], seed=8)
    t0 = time.perf_counter()
    oracle.step_f32(d["x"], d["w"], d["dy"], w["crop"])
    dt = time.perf_counter() - t0
    _ = np
    return nb / dt, cores, f"{nb} images of the headline shape, fwd+bwd_data+bwd_filter fp64 direct, {dt:.1f} s"


# ------------------------------------------------------------------ reference arm
def run_reference(args, w):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    from workloads import make_inputs
    cores = oracle.max_threads()
    per_step = max(1, args.ref_images)
    d = make_inputs(per_step, w["C"], w["K"], w["N"], w["n"], w["crop"], seed=9)
    for _ in range(args.warmup):
        oracle.step_f32(d["x"], d["w"], d["dy"], w["crop"])
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.step_f32(d["x"], d["w"], d["dy"], w["crop"])
    dt = time.perf_counter() - t0
    rate = per_step * args.steps / dt
    sample = f"{per_step} image(s) per step of the headline shape, fp64 direct oracle on {cores} host threads"
    line = {"impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded uniform [-1,1))",
            "config": {"workload": workload_name(w) + " (bounded CPU sample)", "images_per_step": per_step},
            "cpu_baseline": {"value": rate, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm
def run_ours(args, w):
    import torch
    import torch.distributed as dist

    import paper_1601_06815_b200 as oaa

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    B, C, K, N, n, crop = w["B"], w["C"], w["K"], w["N"], w["n"], w["crop"]
    M = out_size(N, n, crop)
    # seeded synthetic inputs, one shard per rank (uniform [-1,1))
    g = torch.Generator(device=dev)
    g.manual_seed(12345 + rank)
    x = torch.rand((B, C, N, N), generator=g, device=dev) * 2 - 1
    wt = torch.rand((K, C, n, n), generator=torch.Generator(device=dev).manual_seed(777), device=dev) * 2 - 1
    dy = torch.rand((B, K, M, M), generator=g, device=dev) * 2 - 1
    y = torch.empty((B, K, M, M), device=dev)
    dx = torch.empty((B, C, N, N), device=dev)
    dw = torch.empty((K, C, n, n), device=dev)
    stream = torch.cuda.current_stream(dev)

    side = torch.cuda.Stream(dev)

    def step():
        # the two backward convolutions are independent: bwd_filter and the
        # dW all-reduce run on a side stream, concurrent with bwd_data
        oaa.conv_fwd(x, wt, crop, out=y)
        side.wait_stream(stream)
        oaa.conv_bwd_filter(x, dy, n, crop, out=dw, stream=side)
        if world > 1:
            with torch.cuda.stream(side):
                dist.all_reduce(dw)
        oaa.conv_bwd_data(dy, wt, N, crop, out=dx)
        stream.wait_stream(side)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    oaa.profile_collect()  # clear
    oaa.profile_enable(True)
    launches0 = oaa.launch_count()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
    oaa.profile_enable(False)
    launches = oaa.launch_count() - launches0
    ms_total = ev0.elapsed_time(ev1)
    kern_ms, kern_cnt = oaa.profile_collect()
    if world > 1:
        t = torch.tensor([ms_total], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    ms_step = ms_total / args.steps
    value = world * B * args.steps / (ms_total / 1e3)

    # e2e through the public API from pinned host buffers (paper_1601_06815_b200.pipeline:
    # chunked H2D / compute / D2H on three streams; bwd_filter over the whole batch)
    e2e = None
    if not args.no_e2e:
        from paper_1601_06815_b200.pipeline import HostStep
        hs = HostStep(B, C, K, N, n, crop, dev, chunks=args.e2e_chunks)
        hx = x.cpu().pin_memory(); hw = wt.cpu().pin_memory(); hdy = dy.cpu().pin_memory()
        hy = torch.empty((B, K, M, M)).pin_memory()
        hdx = torch.empty((B, C, N, N)).pin_memory()
        hdw = torch.empty((K, C, n, n)).pin_memory()

        def e2e_step():
            hs(hx, hw, hdy, hy, hdx, hdw, stream=stream)
            if world > 1:
                dist.all_reduce(hs.dw)

        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ne = max(1, min(args.steps, 5))
        for _ in range(ne):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        ems = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ems], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": world * B * ne / (ems / 1e3), "unit": UNIT, "h2d_bytes_per_step": hs.h2d_bytes,
               "d2h_bytes_per_step": hs.d2h_bytes, "chunks": len(hs.chunks)}

    # roofline of the dominant kernel
    terms = algorithmic_terms(w)
    # the roofline is reported for the fwd op: the largest op that runs alone in the step
    # (bwd_data and bwd_filter overlap on two streams, so their event spans are shared)
    dom = "fwd"
    avg_ms = kern_ms[dom] / max(1, kern_cnt[dom])
    peaks, src = measured_peaks()
    sm_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    alu_peak = 2 * SM_COUNT * FP32_LANES_PER_SM * sm_mhz * 1e6 / 1e12  # TFLOP/s
    achieved = terms["flops"][dom] / (avg_ms / 1e3) / 1e12
    hbm_achieved = terms["bytes"][dom] / (avg_ms / 1e3) / 1e9
    traffic = None
    try:  # measured DRAM bytes of this op from the committed ncu capture (profiles/r1_ncu.md)
        with open(os.path.join(ROOT, "profiles", "r1_traffic.json")) as f:
            traffic = json.load(f)[dom]["op_bytes"]
    except Exception:
        pass
    roofline = {"bound": "alu", "kernel": f"oaa {dom} op (all its launches)", "achieved": achieved,
                "peak": alu_peak, "unit": "TFLOP/s", "frac": achieved / alu_peak, "traffic": traffic,
                "traffic_unit": "bytes per launch (ncu dram read+write, profiles/r1_traffic.json)",
                "algorithmic_bytes": terms["bytes"][dom],
                "peak_source": f"fp32 FFMA 148 SM x 128 lanes x 2 x {sm_mhz:.0f} MHz (MEASURED_PEAKS sm_max_mhz, {src})",
                "hbm_achieved_gbs": hbm_achieved, "hbm_peak_gbs": float(peaks.get("hbm_gbs", 6650.0)),
                "hbm_frac": hbm_achieved / float(peaks.get("hbm_gbs", 6650.0)),
                "kernel_ms": {k: kern_ms[k] / max(1, kern_cnt[k]) for k in kern_ms},
                "kernel_share_of_step": {k: (kern_ms[k] / max(1, kern_cnt[k])) / ms_step for k in kern_ms},
                "kernel_ms_note": "per-op CUDA-event spans on each op's stream; bwd_data and bwd_filter run concurrently, so their spans overlap"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        rate, cores, sample = cpu_oracle_rate(w, budget_s=args.cpu_budget)
        cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded uniform [-1,1), on device)",
                "config": {"workload": workload_name(w), "B_per_gpu": B, "global_batch": B * world,
                           "C": C, "K": K, "N": N, "n": n, "crop": crop, "P": 2 * n - 1,
                           "parallelism": f"dp{world}", "l2": "inputs exceed L2 (dy+y = 3.1 GB/step)",
                           "step": "fwd, then bwd_filter (+ NCCL all_reduce(dW) if N>1) on a side stream concurrent with bwd_data"},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
                "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--ref-images", type=int, default=1)
    ap.add_argument("--e2e-chunks", type=int, default=8)
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    w = dict(HEAD)
    if args.impl == "reference":
        return run_reference(args, w)
    return run_ours(args, w)


if __name__ == "__main__":
    sys.exit(main())
