"""Host-buffer training step of the OaA layer with PCIe transfers overlapped with compute.

`HostStep` is the public call for data that lives in (pinned) host memory: it copies the
batch to the device in chunks on a copy stream, runs fwd and bwd_data per chunk on a
compute stream as soon as each chunk has landed, streams y and dx back per chunk on a
third stream, and runs bwd_filter once over the whole batch (dW is a batch sum).  All
convolution work is the library's kernels; torch only provides memory, streams and
events.
"""
from __future__ import annotations

from typing import Optional

import torch

from . import conv_bwd_data, conv_bwd_filter, conv_fwd, out_size


class HostStep:
    def __init__(self, B: int, C: int, K: int, N: int, n: int, crop: str = "valid",
                 device: Optional[torch.device] = None, chunks: int = 8):
        self.B, self.C, self.K, self.N, self.n, self.crop = B, C, K, N, n, crop
        self.M = out_size(N, n, crop)
        dev = torch.device(device or "cuda")
        self.dev = dev
        M = self.M
        self.x = torch.empty((B, C, N, N), device=dev)
        self.w = torch.empty((K, C, n, n), device=dev)
        self.dy = torch.empty((B, K, M, M), device=dev)
        self.y = torch.empty((B, K, M, M), device=dev)
        self.dx = torch.empty((B, C, N, N), device=dev)
        self.dw = torch.empty((K, C, n, n), device=dev)
        chunks = max(1, min(chunks, B))
        bounds = [round(i * B / chunks) for i in range(chunks + 1)]
        self.chunks = [(a, b) for a, b in zip(bounds, bounds[1:]) if b > a]
        self.s_in = torch.cuda.Stream(dev)
        self.s_cmp = torch.cuda.Stream(dev)
        self.s_out = torch.cuda.Stream(dev)
        self.ev_in = [torch.cuda.Event() for _ in self.chunks]
        self.ev_cmp = [torch.cuda.Event() for _ in self.chunks]
        self.ev_w = torch.cuda.Event()
        self.ev_dw = torch.cuda.Event()
        self.ev_done = torch.cuda.Event()

    @property
    def h2d_bytes(self) -> int:
        return 4 * (self.x.numel() + self.w.numel() + self.dy.numel())

    @property
    def d2h_bytes(self) -> int:
        return 4 * (self.y.numel() + self.dx.numel() + self.dw.numel())

    def __call__(self, hx, hw, hdy, hy, hdx, hdw, stream: Optional[torch.cuda.Stream] = None):
        """Enqueue one step; host outputs hy, hdx, hdw are valid after `stream` (default:
        the current stream) reaches the returned point."""
        cur = stream or torch.cuda.current_stream(self.dev)
        for s in (self.s_in, self.s_cmp, self.s_out):
            s.wait_stream(cur)
        with torch.cuda.stream(self.s_in):
            self.w.copy_(hw, non_blocking=True)
            self.ev_w.record(self.s_in)
            for i, (a, b) in enumerate(self.chunks):
                self.x[a:b].copy_(hx[a:b], non_blocking=True)
                self.dy[a:b].copy_(hdy[a:b], non_blocking=True)
                self.ev_in[i].record(self.s_in)
        self.s_cmp.wait_event(self.ev_w)
        for i, (a, b) in enumerate(self.chunks):
            self.s_cmp.wait_event(self.ev_in[i])
            conv_fwd(self.x[a:b], self.w, self.crop, out=self.y[a:b], stream=self.s_cmp)
            conv_bwd_data(self.dy[a:b], self.w, self.N, self.crop, out=self.dx[a:b], stream=self.s_cmp)
            self.ev_cmp[i].record(self.s_cmp)
            self.s_out.wait_event(self.ev_cmp[i])
            with torch.cuda.stream(self.s_out):
                hy[a:b].copy_(self.y[a:b], non_blocking=True)
                hdx[a:b].copy_(self.dx[a:b], non_blocking=True)
        conv_bwd_filter(self.x, self.dy, self.n, self.crop, out=self.dw, stream=self.s_cmp)
        self.ev_dw.record(self.s_cmp)
        self.s_out.wait_event(self.ev_dw)
        with torch.cuda.stream(self.s_out):
            hdw.copy_(self.dw, non_blocking=True)
        self.ev_done.record(self.s_out)
        cur.wait_event(self.ev_done)
