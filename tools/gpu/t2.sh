#!/bin/bash
out=gpurun_out/t2; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "oas or prepared" > $out/p1.log 2>&1; echo "rc=$?" >> $out/p1.log
timeout 600 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -k "oas" > $out/p2.log 2>&1; echo "rc=$?" >> $out/p2.log
python - >> $out/time.txt 2>&1 <<'PY'
import sys, torch; sys.path.insert(0, '.')
import paper_1601_06815_b200 as oaa
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.rand((128, 3, 224, 224), generator=g, device="cuda") * 2 - 1
w = torch.rand((64, 3, 8, 8), generator=g, device="cuda") * 2 - 1
for name, f in [("oaa", lambda: oaa.conv_fwd(x, w)), ("oas", lambda: oaa.conv_fwd_oas(x, w))]:
    for _ in range(3): f()
    torch.cuda.synchronize()
    oaa.profile_enable(True); oaa.profile_collect_kernels()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10): f()
    b.record(); torch.cuda.synchronize(); oaa.profile_enable(False)
    print(name, a.elapsed_time(b) / 10, {k: v / 10 for k, v in oaa.profile_collect_kernels()[0].items()})
PY
tail -3 $out/p1.log $out/p2.log; cat $out/time.txt
