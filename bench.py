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
  roofline  the dominant kernel (largest CUDA-event time of a serialized pass run right
            after the timed region; its time is the timed region's own span when it runs
            alone there, as the fwd kernels do): its algorithmic work (tools/roofline.py,
            SURVEY.md §8(d)) ÷ its average launch duration, against the measured peak of
            the resource that bounds it (T_roof = max(T_HBM, T_ALU, T_TC)).  `ops` gives
            the same per op and `step_frac` = Σ_op T_roof / ms_per_step.
  cfg5      BASELINE.json configs[4] as north_star states it: global B = 1024 strong-scaled
            over the N ranks (B/N each), fwd → fused backward (dx, dW) → all_reduce(dW),
            with the all-reduce time.
  cpu_baseline  the CPU float64 oracle (direct definition) on the host cores (all and
            one), on a bounded sample of the same workload.
--impl reference runs that oracle as the reference arm (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from tools import roofline as rl  # noqa: E402

HEAD = dict(name="headline", B=128, C=3, K=64, N=224, n=8, crop="valid")
CFG5 = dict(name="sharded", B=1024, C=64, K=128, N=224, n=8, crop="valid")
METRIC = "OaA conv fwd+bwd images/s at N=224,n=8,C=3,K=64; % of HBM/tensor roofline"
UNIT = "images/s"
OPS = ("fwd", "bwd_data", "bwd_filter")


def workload_name(w, per_gpu=True):
    return (f"{w['name']} N={w['N']} n={w['n']} C={w['C']} K={w['K']} B={w['B']}"
            f"{'/gpu' if per_gpu else ' global'} crop={w['crop']}")


# ------------------------------------------------------------------ clocks sampler
class ClockSampler:
    """SM clock + throttle reasons sampled every `period_ms` through NVML while the
    timed region runs (falls back to nvidia-smi -lms)."""
    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, index=0, period_ms=5):
        self.index, self.period_ms = index, period_ms
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))

            def loop():
                while not self._stop.is_set():
                    try:
                        self.samples.append(float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
                        r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        for nm, bit in self.REASONS.items():
                            if r & bit:
                                self.reasons.add(nm)
                    except Exception:
                        pass
                    time.sleep(self.period_ms / 1e3)
            self.t = threading.Thread(target=loop, daemon=True)
            self.t.start()
        except Exception:
            self.t = None
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.t is not None:
            self.t.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"], "samples": 0}
        s = sorted(self.samples)
        return {"sm_mhz": s[len(s) // 2], "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(s), "source": "NVML every 5 ms during the timed region"}


# ------------------------------------------------------------------ CPU oracle timing
def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def cpu_oracle_rate(w, budget_s=15.0, max_images=512):
    """The float64 direct oracle (fwd + bwd_data + bwd_filter) on a sub-batch of the
    workload, on all host cores and on one core."""
    import oracle
    from workloads import make_inputs
    cores = oracle.max_threads()
    d = make_inputs(1, w["C"], w["K"], w["N"], w["n"], w["crop"], seed=7)
    t0 = time.perf_counter()
    oracle.step_f32(d["x"], d["w"], d["dy"], w["crop"], nthreads=1)
    t_one = time.perf_counter() - t0
    nb = int(max(1, min(max_images, budget_s * cores / max(t_one, 1e-3))))
    d = make_inputs(nb, w["C"], w["K"], w["N"], w["n"], w["crop"], seed=8)
    t0 = time.perf_counter()
    oracle.step_f32(d["x"], d["w"], d["dy"], w["crop"], nthreads=cores)
    dt = time.perf_counter() - t0
    return {"value": nb / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{nb} images of the headline shape, fwd+bwd_data+bwd_filter fp64 direct "
                      f"(oracle/oracle.c, OpenMP), {dt:.1f} s on {cores} threads",
            "value_1thread": 1.0 / t_one, "sample_1thread": f"1 image on 1 thread, {t_one:.2f} s",
            "cpu_model": cpu_model(), "os_cpu_count": os.cpu_count()}


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
        oracle.step_f32(d["x"], d["w"], d["dy"], w["crop"], nthreads=cores)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.step_f32(d["x"], d["w"], d["dy"], w["crop"], nthreads=cores)
    dt = time.perf_counter() - t0
    rate = per_step * args.steps / dt
    sample = f"{per_step} image(s) per step of the headline shape, fp64 direct oracle on {cores} host threads"
    line = {"impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded uniform [-1,1))",
            "config": {"workload": workload_name(w) + " (bounded CPU sample)", "images_per_step": per_step},
            "cpu_baseline": {"value": rate, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample,
                             "cpu_model": cpu_model()},
            "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm
def _inputs(torch, dev, B, C, K, N, n, crop, seed):
    """Seeded uniform [-1,1) fp32 drawn on the device (SURVEY.md §8(d) recipe)."""
    M = rl.out_size(N, n, crop)
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    x = torch.rand((B, C, N, N), generator=g, device=dev).mul_(2).sub_(1)
    wt = torch.rand((K, C, n, n), generator=torch.Generator(device=dev).manual_seed(777), device=dev).mul_(2).sub_(1)
    dy = torch.rand((B, K, M, M), generator=g, device=dev).mul_(2).sub_(1)
    return x, wt, dy


class Step:
    """fwd, then bwd_filter (+ all_reduce(dW) when world > 1) on a side stream concurrent
    with bwd_data: the two backward convolutions of PAPER.md:89 are independent."""

    def __init__(self, torch, dist, oaa, dev, world, x, wt, dy, N, n, crop, fused=False):
        self.t, self.dist, self.oaa, self.world, self.fused = torch, dist, oaa, world, fused
        self.x, self.wt, self.dy, self.N, self.n, self.crop = x, wt, dy, N, n, crop
        B, C = x.shape[:2]
        K, M = dy.shape[1], dy.shape[-1]
        self.y = torch.empty((B, K, M, M), device=dev)
        self.dx = torch.empty_like(x)
        self.dw = torch.empty_like(wt)
        self.stream = torch.cuda.current_stream(dev)
        self.side = torch.cuda.Stream(dev)
        self.ar_ev = []

    def __call__(self, time_allreduce=False):
        oaa, t = self.oaa, self.t
        oaa.conv_fwd(self.x, self.wt, self.crop, out=self.y)
        if self.fused:
            # one call for both backward convolutions (NEXT-1: on the tensor-core path the
            # dy spectra are computed once for both GEMMs), then the dW all-reduce
            oaa.conv_bwd(self.x, self.dy, self.wt, self.crop, dx=self.dx, dw=self.dw)
            if self.world > 1:
                if time_allreduce:
                    a, b = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
                    a.record(self.stream)
                self.dist.all_reduce(self.dw)
                if time_allreduce:
                    b.record(self.stream)
                    self.ar_ev.append((a, b))
            return
        self.side.wait_stream(self.stream)
        oaa.conv_bwd_filter(self.x, self.dy, self.n, self.crop, out=self.dw, stream=self.side)
        if self.world > 1:
            with t.cuda.stream(self.side):
                if time_allreduce:
                    a, b = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
                    a.record(self.side)
                self.dist.all_reduce(self.dw)
                if time_allreduce:
                    b.record(self.side)
                    self.ar_ev.append((a, b))
        oaa.conv_bwd_data(self.dy, self.wt, self.N, self.crop, out=self.dx)
        self.stream.wait_stream(self.side)


def _max_over_ranks(torch, dist, world, dev, v):
    if world == 1:
        return v
    t = torch.tensor([v], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _timed(torch, dist, world, dev, fn, steps, stream):
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    return _max_over_ranks(torch, dist, world, dev, e0.elapsed_time(e1))


def run_cfg5(args, torch, dist, oaa, dev, world, rank):
    """BASELINE configs[4] strong-scaled: global B = 1024 split over the ranks."""
    w = dict(CFG5)
    from paper_1601_06815_b200.dist import shard_range
    a, b = shard_range(w["B"], rank, world)
    Bl = b - a
    x, wt, dy = _inputs(torch, dev, Bl, w["C"], w["K"], w["N"], w["n"], w["crop"], seed=4242 + rank)
    st = Step(torch, dist, oaa, dev, world, x, wt, dy, w["N"], w["n"], w["crop"], fused=True)
    for _ in range(3):
        st()
    oaa.profile_collect()
    oaa.profile_enable(True)
    steps = args.cfg5_steps
    ms = _timed(torch, dist, world, dev, lambda: st(time_allreduce=True), steps, st.stream)
    oaa.profile_enable(False)
    oaa.profile_collect()
    k_ms, _ = oaa.profile_collect_kernels()
    ar_ms = None
    if st.ar_ev:
        ar_ms = _max_over_ranks(torch, dist, world, dev, sum(e0.elapsed_time(e1) for e0, e1 in st.ar_ev) / len(st.ar_ev))
    ms_step = ms / steps
    roof_ms = sum(rl.t_roof(rl.op_work(op, Bl, w["C"], w["K"], w["N"], w["n"], w["crop"]))[0] for op in OPS) * 1e3
    rec = {"workload": workload_name(w, per_gpu=False), "global_batch": w["B"], "B_per_gpu": Bl, "n_gpus": world,
           "scaling": "strong", "steps": steps, "warmup": 3, "ms_per_step": ms_step,
           "value": w["B"] / (ms_step / 1e3), "unit": UNIT,
           "tflop_eq_per_s": rl.direct_flops(w["B"], w["C"], w["K"], w["N"], w["n"], w["crop"]) / (ms_step / 1e3) / 1e12,
           "kernels_ms_per_step": {k: v / steps for k, v in k_ms.items()},
           "allreduce_ms": ar_ms, "allreduce_bytes": 4 * w["K"] * w["C"] * w["n"] ** 2,
           "t_roof_ms_per_gpu": roof_ms, "step_frac": roof_ms / ms_step,
           "step": "fwd, then the fused backward (oaa_conv_bwd: dy spectra shared by the bwd_data and bwd_filter GEMMs), then NCCL all_reduce(dW) (N>1)"}
    del st, x, wt, dy
    torch.cuda.empty_cache()
    return rec


def run_ours(args, w):
    import datetime

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
    nccl = None
    if world > 1:
        # communicator logging to a file (stdout carries only the JSON line), bounded
        # collectives, async error handling (torch default TORCH_NCCL_ASYNC_ERROR_HANDLING)
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT,COLL")
        os.environ.setdefault("NCCL_DEBUG_FILE", f"/tmp/oaa_nccl.{os.getpid()}.log")
        os.environ.setdefault("TORCH_NCCL_ASYNC_ERROR_HANDLING", "1")
        dist.init_process_group("nccl", device_id=dev, timeout=datetime.timedelta(minutes=10))
        nccl = {"backend": dist.get_backend(), "comm_nranks": dist.get_world_size(),
                "nccl_version": ".".join(map(str, torch.cuda.nccl.version())),
                "log": os.environ.get("NCCL_DEBUG_FILE")}

    B, C, K, N, n, crop = w["B"], w["C"], w["K"], w["N"], w["n"], w["crop"]
    M = rl.out_size(N, n, crop)
    x, wt, dy = _inputs(torch, dev, B, C, K, N, n, crop, seed=12345 + rank)
    st = Step(torch, dist, oaa, dev, world, x, wt, dy, N, n, crop)
    stream = st.stream

    for _ in range(args.warmup):
        st()
    torch.cuda.synchronize(dev)
    oaa.profile_collect()
    oaa.profile_collect_kernels()  # clear
    oaa.profile_enable(True)
    launches0 = oaa.launch_count()
    with ClockSampler(local) as clk:
        ms_total = _timed(torch, dist, world, dev, st, args.steps, stream)
    oaa.profile_enable(False)
    launches = oaa.launch_count() - launches0
    op_ms, op_cnt = oaa.profile_collect()
    k_ms, k_cnt = oaa.profile_collect_kernels()
    ms_step = ms_total / args.steps
    value = world * B * args.steps / (ms_total / 1e3)

    # ---- roofline: the dominant kernel.  In the timed step bwd_data and bwd_filter run
    # concurrently, so their CUDA-event spans include each other's time; a short
    # serialized pass (same inputs, every op on one stream, right after the timed region)
    # gives every kernel's solo duration -- the share ncu's serialized launch list shows --
    # and picks the dominant kernel.  Its `kernel_ms` is the timed-region span when it ran
    # alone there (the fwd kernels), else the serialized one.
    per_step = {k: v / args.steps for k, v in k_ms.items()}
    fwd_solo = {"spectrum", "xspec", "walk"}  # launched before the backward fork
    oaa.profile_enable(True)
    nser = 3
    for _ in range(nser):
        oaa.conv_fwd(x, wt, crop, out=st.y)
        oaa.conv_bwd_filter(x, dy, n, crop, out=st.dw)
        oaa.conv_bwd_data(dy, wt, N, crop, out=st.dx)
    torch.cuda.synchronize(dev)
    oaa.profile_enable(False)
    oaa.profile_collect()
    s_ms, s_cnt = oaa.profile_collect_kernels()
    serial = {k: v / nser for k, v in s_ms.items()}
    # the overlap-and-save forward (NEXT-2) beside the OaA forward, same inputs, for context
    # (the step itself is OaA, the paper's method)
    def _fwd_ms(f):
        f()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(nser):
            f()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        return e0.elapsed_time(e1) / nser
    variants = {"fwd_overlap_and_add_ms": _fwd_ms(lambda: oaa.conv_fwd(x, wt, crop, out=st.y)),
                "fwd_overlap_and_save_ms": _fwd_ms(lambda: oaa.conv_fwd_oas(x, wt, crop, out=st.y))}
    dom = max(serial, key=serial.get)
    kernel_op = {"walk": "fwd", "xspec": "fwd", "bwdd": "bwd_data", "bwdf": "bwd_filter",
                 "xspec_win": "bwd_filter", "finalize": "bwd_filter", "spectrum": "fwd"}
    dom_op = kernel_op.get(dom, "fwd")
    if dom in fwd_solo and dom in k_ms:
        avg_s, launches_per_step, src_t = k_ms[dom] / k_cnt[dom] / 1e3, k_cnt[dom] / args.steps, "timed region"
    else:
        avg_s, launches_per_step, src_t = s_ms[dom] / s_cnt[dom] / 1e3, s_cnt[dom] / nser, "serialized pass"
    work = rl.kernel_work(dom, dom_op, B, C, K, N, n, crop)
    if launches_per_step != 1:
        work = {q: v / launches_per_step for q, v in work.items()}
    roofline = rl.roofline_record(work, avg_s)
    roofline["kernel"] = f"oaa {dom} ({dom_op})"
    roofline["kernel_ms_source"] = src_t
    roofline["kernels_ms_serialized"] = serial
    roofline["kernel_share_serialized"] = {k: v / sum(serial.values()) for k, v in serial.items()}
    traffic = None
    try:  # ncu dram bytes of this kernel (one --set full capture, profiles/r02_traffic.json)
        with open(os.path.join(ROOT, "profiles", "r02_traffic.json")) as f:
            traffic = json.load(f)["kernels"][dom]["dram_bytes"]
    except Exception:
        pass
    roofline["traffic"] = traffic
    roofline["traffic_source"] = "ncu --set full dram__bytes_read.sum + dram__bytes_write.sum, profiles/r02_traffic.json"
    roofline["kernels_ms_in_step"] = per_step
    roofline["kernels_ms_in_step_note"] = "timed-region event spans; bwd kernels overlap each other"
    ops = {}
    roof_sum = 0.0
    for op in OPS:
        T, bound, terms = rl.t_roof(rl.op_work(op, B, C, K, N, n, crop))
        t = op_ms[op] / max(1, op_cnt[op])
        roof_sum += T * 1e3
        ops[op] = {"ms": t, "t_roof_ms": T * 1e3, "bound": bound, "frac": T * 1e3 / t,
                   "terms_ms": {k: v * 1e3 for k, v in terms.items()}}
    roofline["ops"] = ops
    roofline["ops_note"] = ("per-op CUDA-event spans on each op's stream; bwd_data and bwd_filter run "
                            "concurrently, so their spans overlap")
    roofline["step_t_roof_ms"] = roof_sum
    roofline["step_frac"] = roof_sum / ms_step

    # ---- e2e through the public API from pinned host buffers (paper_1601_06815_b200.pipeline:
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
        ne = max(1, min(args.steps, 5))
        ems = _timed(torch, dist, world, dev, e2e_step, ne, stream)
        e2e = {"value": world * B * ne / (ems / 1e3), "unit": UNIT, "h2d_bytes_per_step": hs.h2d_bytes,
               "d2h_bytes_per_step": hs.d2h_bytes, "chunks": len(hs.chunks)}
        del hs, hx, hw, hdy, hy, hdx, hdw

    del st
    torch.cuda.empty_cache()
    cfg5 = None
    if not args.no_cfg5:
        cfg5 = run_cfg5(args, torch, dist, oaa, dev, world, rank)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_oracle_rate(w, budget_s=args.cpu_budget)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded uniform [-1,1), drawn on device)",
                "config": {"workload": workload_name(w), "B_per_gpu": B, "global_batch": B * world,
                           "C": C, "K": K, "N": N, "n": n, "crop": crop, "P": 2 * n - 1,
                           "parallelism": f"dp{world}", "l2": "inputs exceed L2 (dy+y = 3.1 GB/step)",
                           "step": "fwd, then bwd_filter (+ NCCL all_reduce(dW) if N>1) on a side stream concurrent with bwd_data"},
                "tflop_eq_per_s": world * rl.direct_flops(B, C, K, N, n, crop) / (ms_step / 1e3) / 1e12,
                "roofline": roofline, "variants": variants, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
                "clocks": clk.summary(), "cfg5": cfg5, "nccl": nccl}
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
    ap.add_argument("--no-cfg5", action="store_true")
    ap.add_argument("--cfg5-steps", type=int, default=3)
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
