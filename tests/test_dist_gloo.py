"""World-size-2 gloo test of the batch-sharded step's host logic (SURVEY.md §4 plan item
3): each rank takes its contiguous batch slice, the weight gradient is summed with
all_reduce, and the result must equal the full-batch gradient.  The convolution ops are
a CPU test double built on the float64 oracle -- never a product path."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1601_06815_b200.dist import ConvOps, data_parallel_step, shard_range


def test_shard_range_partitions():
    for B in (0, 1, 5, 128, 1024):
        for world in (1, 2, 3, 8):
            parts = [shard_range(B, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == B
            for (a, b), (c, d) in zip(parts, parts[1:]):
                assert b == c and b - a >= d - c >= b - a - 1
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def _oracle_ops():
    import oracle

    def fwd(x, w, crop):
        return torch.from_numpy(oracle.conv_fwd(x.numpy(), w.numpy(), crop))

    def bwd_data(dy, w, N, crop):
        return torch.from_numpy(oracle.conv_bwd_data(dy.numpy(), w.numpy(), N, crop))

    def bwd_filter(x, dy, n, crop):
        return torch.from_numpy(oracle.conv_bwd_filter(x.numpy(), dy.numpy(), n, crop))

    return ConvOps(fwd, bwd_data, bwd_filter)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from workloads import make_inputs
    d = make_inputs(5, 2, 3, 12, 3, "valid", seed=21)
    a, b = shard_range(5, rank, world)
    x = torch.from_numpy(d["x"][a:b]).double()
    w = torch.from_numpy(d["w"]).double()
    dy = torch.from_numpy(d["dy"][a:b]).double()
    y, dx, dw = data_parallel_step(x, w, dy, "valid", ops=_oracle_ops())
    q.put((rank, a, b, y.numpy(), dx.numpy(), dw.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_gloo_step_matches_full_batch():
    import oracle
    from workloads import make_inputs
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world = 2
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    d = make_inputs(5, 2, 3, 12, 3, "valid", seed=21)
    y_full = oracle.conv_fwd(d["x"], d["w"], "valid")
    dx_full = oracle.conv_bwd_data(d["dy"], d["w"], 12, "valid")
    dw_full = oracle.conv_bwd_filter(d["x"], d["dy"], 3, "valid")
    for rank, a, b, y, dx, dw in res:
        np.testing.assert_allclose(y, y_full[a:b], atol=1e-12)
        np.testing.assert_allclose(dx, dx_full[a:b], atol=1e-12)
        np.testing.assert_allclose(dw, dw_full, atol=1e-11)   # all-reduced = full-batch gradient
