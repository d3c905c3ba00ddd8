"""Batch-sharded data parallelism for the OaA layer.

fwd and bwd_data are independent per image, so each rank processes a contiguous slice
of the global batch with no communication; the only exchange is the sum of the weight
gradient over ranks (one all-reduce of K·C·n² floats), issued right after bwd_filter
so it overlaps bwd_data on the stream.

The convolution ops are injectable (`ops`) so the sharding / reduction logic can be
exercised on CPU with the gloo backend in tests; the default ops are the CUDA library.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional, Tuple

import torch
import torch.distributed as dist


def shard_range(global_batch: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous [start, stop) slice of the batch owned by `rank` (sizes differ by ≤ 1)."""
    if world < 1 or not (0 <= rank < world) or global_batch < 0:
        raise ValueError("bad shard arguments")
    base, rem = divmod(global_batch, world)
    start = rank * base + min(rank, rem)
    return start, start + base + (1 if rank < rem else 0)


@dataclass
class ConvOps:
    fwd: Callable
    bwd_data: Callable
    bwd_filter: Callable


def cuda_ops() -> ConvOps:
    from . import conv_bwd_data, conv_bwd_filter, conv_fwd
    return ConvOps(conv_fwd, conv_bwd_data, conv_bwd_filter)


def data_parallel_step(x: torch.Tensor, w: torch.Tensor, dy: torch.Tensor, crop: str = "valid",
                       ops: Optional[ConvOps] = None, group=None, average: bool = False):
    """One training step of the layer on this rank's shard: y = fwd(x, w),
    dw = all_reduce(bwd_filter(x, dy)), dx = bwd_data(dy, w).  Returns (y, dx, dw)."""
    ops = ops or cuda_ops()
    N, n = x.shape[-1], w.shape[-1]
    y = ops.fwd(x, w, crop)
    dw = ops.bwd_filter(x, dy, n, crop)
    work = None
    if dist.is_available() and dist.is_initialized():
        work = dist.all_reduce(dw, op=dist.ReduceOp.SUM, group=group, async_op=True)
    dx = ops.bwd_data(dy, w, N, crop)
    if work is not None:
        work.wait()
        if average:
            dw /= dist.get_world_size(group)
    return y, dx, dw
