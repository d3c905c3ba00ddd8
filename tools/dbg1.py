import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, oracle, paper_1601_06815_b200 as oaa
from workloads import make_inputs
for (N, n, crop) in [(1, 5, "full"), (3, 5, "full"), (7, 3, "valid"), (20, 8, "same")]:
    for (B, C, K) in [(1, 1, 1), (2, 3, 2), (3, 2, 3)]:
        d = make_inputs(B, C, K, N, n, crop, seed=N * 100 + n * 7 + B)
        dy = torch.from_numpy(d["dy"]).cuda(); w = torch.from_numpy(d["w"]).cuda()
        x = torch.from_numpy(d["x"]).cuda()
        dx = oaa.conv_bwd_data(dy, w, N, crop).cpu().numpy()
        ref = oracle.conv_bwd_data(d["dy"], d["w"], N, crop)
        y = oaa.conv_fwd(x, w, crop).cpu().numpy(); refy = oracle.conv_fwd(d["x"], d["w"], crop)
        e = np.abs(dx - ref).max(); ey = np.abs(y - refy).max()
        print(N, n, crop, (B, C, K), "dx err", e, "y err", ey)
        if e > 1e-4: print("got", dx.ravel()[:8], "\nref", ref.ravel()[:8])
