#!/bin/bash
# GPU-box probe: host CPU, measured compute peaks, oracle throughput at full size.
set -x
mkdir -p gpurun_out/probe
lscpu | head -20 > gpurun_out/probe/lscpu.txt; nproc >> gpurun_out/probe/lscpu.txt
nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/microbench/peaks.cu -o /tmp/peaks && \
  for i in 1 2 3; do /tmp/peaks; done > gpurun_out/probe/peaks.jsonl 2>&1
python - <<'PY' > gpurun_out/probe/oracle_time.txt 2>&1
import time, numpy as np, sys
sys.path.insert(0, '.')
import oracle
from workloads import make_inputs
for B in (4, 16):
    d = make_inputs(B, 3, 64, 224, 8, "valid", seed=1)
    t=time.time(); oracle.conv_fwd(d["x"], d["w"], "valid"); t1=time.time()-t
    t=time.time(); oracle.conv_bwd_data(d["dy"], d["w"], 224, "valid"); t2=time.time()-t
    t=time.time(); oracle.conv_bwd_filter(d["x"], d["dy"], 8, "valid"); t3=time.time()-t
    print("B", B, "fwd", t1, "bwdd", t2, "bwdf", t3, "threads", oracle.max_threads(), flush=True)
PY
cat gpurun_out/probe/*
