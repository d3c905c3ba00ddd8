"""Time fwd / bwd_data / bwd_filter (CUDA events, median of reps) for the library at
$OAA_LIB (default in-tree).  usage: python tools/time_ops.py [B,C,K,N,n] [crop]"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1601_06815_b200 as oaa
B, C, K, N, n = 128, 3, 64, 224, 8
if len(sys.argv) > 1:
    B, C, K, N, n = map(int, sys.argv[1].split(","))
crop = sys.argv[2] if len(sys.argv) > 2 else "valid"
M = oaa.out_size(N, n, crop)
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.rand((B, C, N, N), generator=g, device="cuda") * 2 - 1
w = torch.rand((K, C, n, n), generator=g, device="cuda") * 2 - 1
dy = torch.rand((B, K, M, M), generator=g, device="cuda") * 2 - 1
y = torch.empty((B, K, M, M), device="cuda"); dx = torch.empty_like(x); dw = torch.empty_like(w)
ops = {"fwd": lambda: oaa.conv_fwd(x, w, crop, out=y),
       "bwd_data": lambda: oaa.conv_bwd_data(dy, w, N, crop, out=dx),
       "bwd_filter": lambda: oaa.conv_bwd_filter(x, dy, n, crop, out=dw),
       "bwd_fused": lambda: oaa.conv_bwd(x, dy, w, crop)}
res = {}
for name, f in ops.items():
    for _ in range(3): f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(7):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); f(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    ts.sort(); res[name] = round(ts[len(ts) // 2], 4)
res["lib"] = os.environ.get("OAA_LIB", "in-tree")
print(json.dumps(res))
