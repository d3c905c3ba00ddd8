"""Per-kernel CUDA-event breakdown of each op (library profiling hook), serialized.
usage: python tools/kernel_breakdown.py B,C,K,N,n [crop] [reps]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1601_06815_b200 as oaa
B, C, K, N, n = map(int, sys.argv[1].split(","))
crop = sys.argv[2] if len(sys.argv) > 2 else "valid"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
M = oaa.out_size(N, n, crop)
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.rand((B, C, N, N), generator=g, device="cuda") * 2 - 1
w = torch.rand((K, C, n, n), generator=g, device="cuda") * 2 - 1
dy = torch.rand((B, K, M, M), generator=g, device="cuda") * 2 - 1
y = torch.empty((B, K, M, M), device="cuda"); dx = torch.empty_like(x); dw = torch.empty_like(w)
ops = {"fwd": lambda: oaa.conv_fwd(x, w, crop, out=y),
       "bwd_data": lambda: oaa.conv_bwd_data(dy, w, N, crop, out=dx),
       "bwd_filter": lambda: oaa.conv_bwd_filter(x, dy, n, crop, out=dw)}
out = {"cfg": [B, C, K, N, n, crop]}
for name, f in ops.items():
    f(); torch.cuda.synchronize()
    oaa.profile_enable(True); oaa.profile_collect(); oaa.profile_collect_kernels()
    for _ in range(reps):
        f()
    torch.cuda.synchronize()
    oaa.profile_enable(False)
    op_ms, _ = oaa.profile_collect()
    k_ms, k_cnt = oaa.profile_collect_kernels()
    out[name] = {"op_ms": round(op_ms[name] / reps, 4),
                 "kernels_ms": {k: round(v / reps, 4) for k, v in k_ms.items()},
                 "launches": {k: v // reps for k, v in k_cnt.items()}}
print(json.dumps(out))
