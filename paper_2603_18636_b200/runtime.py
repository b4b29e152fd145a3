"""Streamed execution of the attention layer over host-resident batches.

A serving loop feeds one layer call per denoising step / request with Q, K, V that live in pinned
host memory and reads O back.  `StreamedLayer` overlaps the three phases of consecutive calls on
three CUDA streams with `depth` device buffer sets: the upload of call i+1 (host -> device), the
layer of call i, and the download of call i-1 (device -> host) run concurrently, ordered only by
CUDA events (no host synchronisation inside the loop).  PCIe traffic per call at Wan2.1-14B 720p
is 3 x 774 MB in and 774 MB out, so on one B200 the loop is bound by the host -> device link, not
by the 25 ms layer.

This is plumbing around the public entry point (`coclust_sparse_attention` or any callable with
the same (q, k, v, out=...) contract); every step of the layer itself runs in libcoclust.
"""
from __future__ import annotations

import torch


class StreamedLayer:
    def __init__(self, layer_fn, shape, device, dtype=torch.bfloat16, depth: int = 2):
        """layer_fn(q, k, v, out) enqueues one layer on torch's current stream."""
        self.fn = layer_fn
        self.depth = depth
        dev = torch.device(device)
        self.h2d = torch.cuda.Stream(dev)
        self.comp = torch.cuda.Stream(dev)
        self.d2h = torch.cuda.Stream(dev)
        mk = lambda: torch.empty(shape, dtype=dtype, device=dev)
        self.bufs = [(mk(), mk(), mk(), mk()) for _ in range(depth)]  # q, k, v, out per slot
        ev = lambda: [torch.cuda.Event() for _ in range(depth)]
        self.up_done, self.comp_done, self.down_done = ev(), ev(), ev()
        self.used = [False] * depth

    def submit(self, i: int, hq, hk, hv, ho):
        """Enqueue call i: upload (hq, hk, hv) -> layer -> download into ho (pinned host)."""
        s = i % self.depth
        dq, dk, dv, do = self.bufs[s]
        if self.used[s]:
            self.h2d.wait_event(self.comp_done[s])    # the layer of call i - depth read this slot
        with torch.cuda.stream(self.h2d):
            dq.copy_(hq, non_blocking=True)
            dk.copy_(hk, non_blocking=True)
            dv.copy_(hv, non_blocking=True)
            self.up_done[s].record()
        self.comp.wait_event(self.up_done[s])
        if self.used[s]:
            self.comp.wait_event(self.down_done[s])   # the output of call i - depth was read
        with torch.cuda.stream(self.comp):
            self.fn(dq, dk, dv, do)
            self.comp_done[s].record()
        self.d2h.wait_event(self.comp_done[s])
        with torch.cuda.stream(self.d2h):
            ho.copy_(do, non_blocking=True)
            self.down_done[s].record()
        self.used[s] = True

    def last_event(self, i: int) -> torch.cuda.Event:
        return self.down_done[i % self.depth]
