"""Small calls of every entry point and kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck).  usage: python tools/sanitize_cases.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1601_06815_b200 as oaa
from workloads import make_inputs

CASES = [(2, 3, 8, 40, 8, "valid"),    # walker / bwd_data / bwd_filter SIMT kernels, fused bwd
         (2, 2, 5, 23, 5, "full"),     # n ∤ 32, full crop
         (1, 6, 7, 19, 4, "same"),     # first-generation engine (C > 4, small K)
         (2, 16, 20, 17, 3, "same"),   # tensor-core path (tile spectra, bin GEMM, walker load)
         (2, 32, 32, 32, 8, "valid"),  # tensor-core path with TMA tensor stores of Y-hat
         (1, 2, 3, 12, 1, "valid"),    # n = 1
         (1, 3, 5, 45, 3, "same"),     # blocks b = 16 − n (walker, bwd_data), two stage-B rounds
         (2, 2, 4, 70, 7, "full")]     # b = 9 for n = 7, ragged last block
for (B, C, K, N, n, crop) in CASES:
    d = make_inputs(B, C, K, N, n, crop, seed=3)
    x = torch.from_numpy(d["x"]).cuda(); w = torch.from_numpy(d["w"]).cuda(); dy = torch.from_numpy(d["dy"]).cuda()
    oaa.conv_fwd(x, w, crop)
    oaa.conv_bwd_data(dy, w, N, crop)
    oaa.conv_bwd_filter(x, dy, n, crop)
    oaa.conv_bwd(x, dy, w, crop)
    if C <= 4 or (C >= 16 and K >= 16):
        oaa.conv_fwd_oas(x, w, crop)
    oaa.PreparedWeights(w, N, "fwd", crop).fwd(x)
    torch.cuda.synchronize()
    print("ok", (B, C, K, N, n, crop), flush=True)
