import sys, os
sys.path.insert(0, os.getcwd())
import torch, paper_1601_06815_b200 as oaa
from workloads import make_inputs
d = make_inputs(2, 3, 8, 40, 8, "valid", seed=1)
x = torch.from_numpy(d["x"]).cuda(); w = torch.from_numpy(d["w"]).cuda()
oaa.conv_fwd(x, w, "valid"); torch.cuda.synchronize(); print("ok")
