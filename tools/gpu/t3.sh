#!/bin/bash
out=gpurun_out/t3; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fused or prepared or tensor_core or small_grid" > $out/p1.log 2>&1; echo "rc=$?" >> $out/p1.log
timeout 600 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -k "fused" > $out/p2.log 2>&1; echo "rc=$?" >> $out/p2.log
python - >> $out/time.txt 2>&1 <<'PY'
import sys, torch; sys.path.insert(0, '.')
import paper_1601_06815_b200 as oaa
for (B, C, K, N, n) in [(256, 96, 256, 27, 5), (128, 64, 128, 224, 8), (1024, 64, 128, 224, 8), (128, 3, 64, 224, 8)]:
    M = N - n + 1
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.rand((B, C, N, N), generator=g, device="cuda") * 2 - 1
    w = torch.rand((K, C, n, n), generator=g, device="cuda") * 2 - 1
    dy = torch.rand((B, K, M, M), generator=g, device="cuda") * 2 - 1
    def sep():
        oaa.conv_bwd_filter(x, dy, n); oaa.conv_bwd_data(dy, w, N)
    def fused():
        oaa.conv_bwd(x, dy, w)
    for name, f in [("separate", sep), ("fused", fused)]:
        for _ in range(2): f()
        torch.cuda.synchronize()
        oaa.profile_enable(True); oaa.profile_collect_kernels()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        reps = 2 if B == 1024 else 5
        a.record()
        for _ in range(reps): f()
        b.record(); torch.cuda.synchronize(); oaa.profile_enable(False)
        print((B, C, K, N, n), name, round(a.elapsed_time(b) / reps, 3), {k: round(v / reps, 3) for k, v in oaa.profile_collect_kernels()[0].items()}, flush=True)
    del x, w, dy
    torch.cuda.empty_cache()
PY
tail -n 3 $out/p1.log $out/p2.log; cat $out/time.txt
