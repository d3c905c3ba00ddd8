"""Seeded synthetic workloads shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no convolution, no transform, no
overlap-add).  It only knows the workload shapes of BASELINE.json's configs and
draws seeded inputs, so both sides of every parity check consume the *same* fp32
values (SURVEY.md §8(d) "Inputs": x, w, dy i.i.d. uniform [-1, 1], seeds 0/1/2,
drawn with a CPU torch.Generator; "timing is data-independent").

Output-size bookkeeping (Full / Valid / Same) is the ConvMode *shape* definition of
SPEC.md:188 and is needed here only to size dy; the oracle and the CUDA library each
compute the crop themselves.
"""
from __future__ import annotations

import dataclasses
from typing import Dict, List

import numpy as np
import torch

CROPS = {"full": 0, "valid": 1, "same": 2}


def out_size(N: int, n: int, crop: str) -> int:
    """ConvMode output side: Full N+n-1, Valid N-n+1, Same N."""
    c = crop if isinstance(crop, str) else {v: k for k, v in CROPS.items()}[crop]
    if c == "full":
        return N + n - 1
    if c == "valid":
        return N - n + 1
    if c == "same":
        return N
    raise ValueError(crop)


@dataclasses.dataclass(frozen=True)
class Workload:
    name: str
    B: int
    C: int
    K: int
    N: int
    n: int
    crop: str = "valid"
    passes: tuple = ("fwd", "bwd_data", "bwd_filter")

    @property
    def M(self) -> int:
        return out_size(self.N, self.n, self.crop)


# BASELINE.json "configs" (in order).  Sweep B is unstated in BASELINE.json; SURVEY.md
# §8(d) row 3 fixes it to the headline's 128.
CONFIGS: Dict[str, Workload] = {
    "parity": Workload("parity", B=1, C=1, K=1, N=32, n=3, passes=("fwd",)),
    "headline": Workload("headline", B=128, C=3, K=64, N=224, n=8),
    "alexnet": Workload("alexnet", B=256, C=96, K=256, N=27, n=5),
    "sharded": Workload("sharded", B=1024, C=64, K=128, N=224, n=8),
}
SWEEP: List[Workload] = [
    Workload(f"sweep_N{N}_n{n}", B=128, C=3, K=64, N=N, n=n)
    for N in (16, 32, 64, 128, 224) for n in (3, 5, 7, 8)
]

SEED_X, SEED_W, SEED_DY = 0, 1, 2


def uniform(shape, seed: int) -> np.ndarray:
    """i.i.d. uniform [-1, 1) fp32, drawn with a seeded CPU torch.Generator."""
    g = torch.Generator(device="cpu")
    g.manual_seed(int(seed))
    t = torch.rand(tuple(int(s) for s in shape), generator=g, dtype=torch.float32)
    t.mul_(2.0).sub_(1.0)
    return t.numpy()


def make_inputs(B: int, C: int, K: int, N: int, n: int, crop: str = "valid",
                seed: int = 0) -> Dict[str, np.ndarray]:
    """x[B,C,N,N], w[K,C,n,n], dy[B,K,M,M] (fp32, C-contiguous).

    `seed` offsets the three canonical seeds so tests can draw independent cases.
    """
    M = out_size(N, n, crop)
    return {
        "x": uniform((B, C, N, N), SEED_X + 3 * seed),
        "w": uniform((K, C, n, n), SEED_W + 3 * seed),
        "dy": uniform((B, K, M, M), SEED_DY + 3 * seed),
    }
