"""PCIe floor of the end-to-end metric: pinned host -> device bandwidth for one layer's Q, K, V
(3 x 774 MB at Wan2.1-14B 720p), split over 1-4 streams, and the time of the three uploads with
the 774 MB download of O running concurrently (the per-step floor of a pipelined e2e loop)."""
import time

import torch

n = 774144000 // 2
h = [torch.empty(n, dtype=torch.bfloat16).pin_memory() for _ in range(3)]
d = [torch.empty(n, dtype=torch.bfloat16, device="cuda") for _ in range(3)]
s = [torch.cuda.Stream() for _ in range(4)]
for ns, ch in [(1, 1), (2, 2), (4, 4), (2, 8)]:
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(3):
            for c in range(ch):
                with torch.cuda.stream(s[(i * ch + c) % ns]):
                    lo, hi = c * n // ch, (c + 1) * n // ch
                    d[i][lo:hi].copy_(h[i][lo:hi], non_blocking=True)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
    print(ns, "streams", ch, "chunks per tensor: H2D GB/s %.1f" % (3 * n * 2 / (t1 - t0) / 1e9))
torch.cuda.synchronize()
t0 = time.perf_counter()
with torch.cuda.stream(s[0]):
    for i in range(3):
        d[i].copy_(h[i], non_blocking=True)
with torch.cuda.stream(s[1]):
    h[0].copy_(d[1], non_blocking=True)
torch.cuda.synchronize()
print("3 x H2D + 1 x D2H concurrently: %.1f ms" % ((time.perf_counter() - t0) * 1e3))
