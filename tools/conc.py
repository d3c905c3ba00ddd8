"""Experiment: headline step with bwd_filter on a side stream, concurrent with bwd_data
(and optionally fwd).  usage: python tools/conc.py"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1601_06815_b200 as oaa
B, C, K, N, n, crop = 128, 3, 64, 224, 8, "valid"
M = N - n + 1
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.rand((B, C, N, N), generator=g, device="cuda") * 2 - 1
w = torch.rand((K, C, n, n), generator=g, device="cuda") * 2 - 1
dy = torch.rand((B, K, M, M), generator=g, device="cuda") * 2 - 1
y = torch.empty((B, K, M, M), device="cuda"); dx = torch.empty_like(x); dw = torch.empty_like(w)
main = torch.cuda.current_stream(); side = torch.cuda.Stream(); side2 = torch.cuda.Stream()
def seq():
    oaa.conv_fwd(x, w, crop, out=y); oaa.conv_bwd_filter(x, dy, n, crop, out=dw); oaa.conv_bwd_data(dy, w, N, crop, out=dx)
def conc_bwd():
    oaa.conv_fwd(x, w, crop, out=y)
    side.wait_stream(main)
    oaa.conv_bwd_filter(x, dy, n, crop, out=dw, stream=side)
    oaa.conv_bwd_data(dy, w, N, crop, out=dx)
    main.wait_stream(side)
def conc_all():
    side.wait_stream(main); side2.wait_stream(main)
    oaa.conv_bwd_filter(x, dy, n, crop, out=dw, stream=side)
    oaa.conv_bwd_data(dy, w, N, crop, out=dx, stream=side2)
    oaa.conv_fwd(x, w, crop, out=y)
    main.wait_stream(side); main.wait_stream(side2)
res = {}
for name, f in [("seq", seq), ("conc_bwd", conc_bwd), ("conc_all", conc_all), ("seq2", seq)]:
    for _ in range(3): f()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20): f()
    b.record(); torch.cuda.synchronize()
    res[name] = a.elapsed_time(b) / 20
print(json.dumps(res))
