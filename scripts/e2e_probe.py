"""Where the end-to-end step time goes: the StreamedLayer loop of bench.py's e2e leg with (a) the
real layer, (b) no layer (copies only, same events), (c) the layer alone on device-resident data;
plus the plain copy floor of scripts/h2d_bw.py.  Wan2.1-14B 720p, 40 heads, FIXED 0.2."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2603_18636_b200 as pb
from paper_2603_18636_b200.runtime import StreamedLayer
from synthetic import config_workload

w = config_workload("wan14b_720p", device="cuda")
q, k, v = w.q, w.k, w.v
H = q.shape[1]
budget = torch.full((H,), 0.2, device="cuda")
ws = pb.Workspace()
hq, hk, hv = (t.cpu().pin_memory() for t in (q, k, v))
hos = [torch.empty(q.shape, dtype=q.dtype).pin_memory() for _ in range(2)]


def layer(dq, dk, dv, do):
    pb.coclust_sparse_attention(dq, dk, dv, 100, 500, 2, budget, rule=pb.RULE_FIXED, out=do, ws=ws)


def noop(dq, dk, dv, do):
    pass


def timed(fn, depth, K=8):
    sl = StreamedLayer(fn, q.shape, "cuda", depth=depth)
    for i in range(2):
        sl.submit(i, hq, hk, hv, hos[i % 2])
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(sl.h2d)
    for i in range(K):
        sl.submit(i, hq, hk, hv, hos[i % 2])
    b.record(sl.d2h)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / K


for depth in (2, 3):
    print(f"depth {depth}: layer + copies {timed(layer, depth):.2f} ms/step, copies only {timed(noop, depth):.2f} ms/step", flush=True)
out = torch.empty_like(q)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
layer(q, k, v, out)
torch.cuda.synchronize()
e0.record()
for _ in range(5):
    layer(q, k, v, out)
e1.record()
torch.cuda.synchronize()
print(f"layer alone {e0.elapsed_time(e1) / 5:.2f} ms", flush=True)
