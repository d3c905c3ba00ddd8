#!/bin/bash
out=gpurun_out/t4; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fused or small_grid or largest or channel" > $out/p1.log 2>&1; echo "rc=$?" >> $out/p1.log
python - >> $out/time.txt 2>&1 <<'PY'
import sys, torch; sys.path.insert(0, '.')
import paper_1601_06815_b200 as oaa
for (B, C, K, N, n) in [(128, 3, 64, 224, 8), (128, 3, 64, 224, 5), (128, 3, 64, 224, 3), (128, 3, 64, 64, 8)]:
    M = N - n + 1
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.rand((B, C, N, N), generator=g, device="cuda") * 2 - 1
    w = torch.rand((K, C, n, n), generator=g, device="cuda") * 2 - 1
    dy = torch.rand((B, K, M, M), generator=g, device="cuda") * 2 - 1
    side = torch.cuda.Stream()
    cur = torch.cuda.current_stream()
    def sep():
        oaa.conv_bwd_filter(x, dy, n); oaa.conv_bwd_data(dy, w, N)
    def two_streams():
        side.wait_stream(cur)
        oaa.conv_bwd_filter(x, dy, n, stream=side); oaa.conv_bwd_data(dy, w, N)
        cur.wait_stream(side)
    def fused():
        oaa.conv_bwd(x, dy, w)
    for name, f in [("separate", sep), ("two_streams", two_streams), ("fused", fused)]:
        for _ in range(3): f()
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10): f()
        b.record(); torch.cuda.synchronize()
        print((B, C, K, N, n), name, round(a.elapsed_time(b) / 10, 4), flush=True)
PY
tail -n 3 $out/p1.log; cat $out/time.txt
