"""The per-rank layer of head-parallel Wan2.1-14B 720p at P ranks (its H/P heads, global sampler
streams), timed as CUDA-graph replays; run under ncu for the per-kernel launch list.

    python scripts/few_heads.py [--P 8] [--rank 0] [--steps 20]
"""
import argparse
import sys

import torch

sys.path.insert(0, ".")
import paper_2603_18636_b200 as pb  # noqa: E402
from paper_2603_18636_b200.dist import head_range  # noqa: E402
from synthetic import config_workload  # noqa: E402

def grouped(q, k, v, budget, lo, H, G, wss, outs, streams):
    """The rank's heads in G groups, each its own layer call on its own stream (fork / join with
    events): the clustering of one group can fill SMs the other group's attention leaves idle."""
    Hl = q.shape[1]
    bounds = [round(g * Hl / G) for g in range(G + 1)]
    cur = torch.cuda.current_stream()
    evs = []
    for g in range(G):
        s = streams[g]
        s.wait_stream(cur)
        with torch.cuda.stream(s):
            a, b = bounds[g], bounds[g + 1]
            pb.coclust_sparse_attention(q[:, a:b], k[:, a:b], v[:, a:b], 100, 500, 2, budget[a:b], rule=pb.RULE_FIXED,
                                        out=outs[g], ws=wss[g], head_offset=lo + a, heads_total=H)
            e = torch.cuda.Event()
            e.record(s)
            evs.append(e)
    for e in evs:
        cur.wait_event(e)


ap = argparse.ArgumentParser()
ap.add_argument("--P", type=int, default=8)
ap.add_argument("--rank", type=int, default=0)
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--no-graph", action="store_true")
ap.add_argument("--groups", type=int, default=1, help="head groups on separate streams (fork/join)")
a = ap.parse_args()
w = config_workload("wan14b_720p", device="cuda")
H = w.q.shape[1]
lo, hi = head_range(H, a.P, a.rank)
q, k, v = (t[:, lo:hi].contiguous() for t in (w.q, w.k, w.v))
del w
budget = torch.full((hi - lo,), 0.2, device="cuda")
out = torch.empty_like(q)
ws = pb.Workspace()
if a.groups > 1:
    bounds = [round(g * (hi - lo) / a.groups) for g in range(a.groups + 1)]
    wss = [pb.Workspace() for _ in range(a.groups)]
    outs = [torch.empty_like(q[:, bounds[g]:bounds[g + 1]]) for g in range(a.groups)]
    streams = [torch.cuda.Stream() for _ in range(a.groups)]
    run = lambda: grouped(q, k, v, budget, lo, H, a.groups, wss, outs, streams)
else:
    run = lambda: pb.coclust_sparse_attention(q, k, v, 100, 500, 2, budget, rule=pb.RULE_FIXED, out=out, ws=ws,
                                              head_offset=lo, heads_total=H)
for _ in range(3):
    run()
torch.cuda.synchronize()
if a.no_graph:
    step = run
else:
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        run()
    torch.cuda.current_stream().wait_stream(s)
    with torch.cuda.graph(g):
        run()
    step = g.replay
for _ in range(3):
    step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.steps):
    step()
e1.record()
torch.cuda.synchronize()
print(f"P={a.P} rank={a.rank} heads={hi - lo} groups={a.groups}: {e0.elapsed_time(e1) / a.steps:.3f} ms per layer")
