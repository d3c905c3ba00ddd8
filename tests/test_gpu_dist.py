"""The batch-sharded training step with the REAL CUDA kernels: two ranks
(both on cuda:0 -- this box has one GPU), gloo all-reduce of dW on CUDA tensors, global
B = 16, each rank's y / dx shard and the all-reduced dW compared element by element
with the float64 oracle on the full batch.  The same `paper_1601_06815_b200.dist`
code runs under NCCL on an 8-GPU node (bench.py --gpus N)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

CASES = [  # (B, C, K, N, n, crop): the headline kernel family and the tensor-core path
    (16, 3, 64, 64, 8, "valid"),
    (16, 16, 24, 30, 5, "same"),
]


def _worker(rank, world, port, case, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_1601_06815_b200.dist import data_parallel_step, shard_range
        from workloads import make_inputs
        B, C, K, N, n, crop = case
        d = make_inputs(B, C, K, N, n, crop, seed=31)
        a, b = shard_range(B, rank, world)
        x = torch.from_numpy(d["x"][a:b]).cuda()
        w = torch.from_numpy(d["w"]).cuda()
        dy = torch.from_numpy(d["dy"][a:b]).cuda()
        y, dx, dw = data_parallel_step(x, w, dy, crop)   # default ops: the CUDA library
        torch.cuda.synchronize()
        q.put((rank, a, b, y.cpu().numpy(), dx.cpu().numpy(), dw.cpu().numpy(), None))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # surface the failure in the parent
        q.put((rank, 0, 0, None, None, None, repr(e)))
        raise


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _check(got, ref, what):
    got = np.asarray(got, dtype=np.float64)
    rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    mx = np.abs(got - ref).max() / np.abs(ref).max()
    assert rel <= 1e-5 and mx <= 1e-4, f"{what}: rel-L2 {rel:.3e}, max {mx:.3e}"


@pytest.mark.parametrize("case", CASES, ids=lambda c: "B{}C{}K{}N{}n{}{}".format(*c))
def test_two_rank_cuda_step_matches_oracle(case):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import oracle
    from workloads import make_inputs
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world, port = 2, _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
    for r in res:
        assert r[6] is None, f"rank {r[0]} failed: {r[6]}"
    assert all(p.exitcode == 0 for p in procs)
    B, C, K, N, n, crop = case
    d = make_inputs(B, C, K, N, n, crop, seed=31)
    y_full = oracle.conv_fwd(d["x"], d["w"], crop)
    dx_full = oracle.conv_bwd_data(d["dy"], d["w"], N, crop)
    dw_full = oracle.conv_bwd_filter(d["x"], d["dy"], n, crop)
    for rank, a, b, y, dx, dw, _ in res:
        _check(y, y_full[a:b], f"rank {rank} y")
        _check(dx, dx_full[a:b], f"rank {rank} dx")
        _check(dw, dw_full, f"rank {rank} all-reduced dw")
