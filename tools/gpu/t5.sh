#!/bin/bash
out=gpurun_out/t5; mkdir -p $out
for lib in in-tree "_build_oaa_exp_fused_slots=74" "_build_oaa_exp_fused_slots=222" "_build_oaa_exp_fused_slots=296"; do
  if [ "$lib" != in-tree ]; then export OAA_LIB=$PWD/paper_1601_06815_b200/$lib/liboaa.so; fi
  python - >> $out/time.txt 2>&1 <<'PY'
import os, sys, torch; sys.path.insert(0, '.')
import paper_1601_06815_b200 as oaa
B, C, K, N, n = 128, 3, 64, 224, 8
M = N - n + 1
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.rand((B, C, N, N), generator=g, device="cuda") * 2 - 1
w = torch.rand((K, C, n, n), generator=g, device="cuda") * 2 - 1
dy = torch.rand((B, K, M, M), generator=g, device="cuda") * 2 - 1
f = lambda: oaa.conv_bwd(x, dy, w)
for _ in range(3): f()
torch.cuda.synchronize()
a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20): f()
b.record(); torch.cuda.synchronize()
print(os.environ.get("OAA_LIB", "in-tree(148)")[-40:], round(a.elapsed_time(b) / 20, 4), flush=True)
PY
done
cat $out/time.txt
