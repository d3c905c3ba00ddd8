"""Run the headline step a few times (for ncu).  usage: python tools/prof_step.py [reps] [ops]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1601_06815_b200 as oaa
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
ops = sys.argv[2].split(",") if len(sys.argv) > 2 else ["fwd", "bwd_data", "bwd_filter"]
B, C, K, N, n = 128, 3, 64, 224, 8
if len(sys.argv) > 3:
    B, C, K, N, n = map(int, sys.argv[3].split(","))
M = N - n + 1
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.rand((B, C, N, N), generator=g, device="cuda") * 2 - 1
w = torch.rand((K, C, n, n), generator=g, device="cuda") * 2 - 1
dy = torch.rand((B, K, M, M), generator=g, device="cuda") * 2 - 1
for _ in range(reps):
    if "fwd" in ops: y = oaa.conv_fwd(x, w)
    if "bwd_data" in ops: dx = oaa.conv_bwd_data(dy, w, N)
    if "bwd_filter" in ops: dw = oaa.conv_bwd_filter(x, dy, n)
torch.cuda.synchronize()
print("ok")
