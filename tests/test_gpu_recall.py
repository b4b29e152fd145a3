"""Matched-budget attention recall of co-clustering vs the independent k-means baseline (P:181-183,
P:1079-1081; R19) on planted-region synthetic attention.

Both partitions come from the library (coclust_assign / kmeans_assign, same sampler and iteration
count); the dense attention, the high-attention reference set and the recall are the oracle's.
Set RECALL_OUT=path to write the comparison as JSON (profiles/r01_recall.json).
"""
import json
import math
import os

import numpy as np
import pytest
import torch

from oracle import svoo
from synthetic import video_qkv

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pb():
    from paper_2603_18636_b200 import build
    build.build()
    import paper_2603_18636_b200 as m
    m.lib()
    return m


def f64(t):
    return t.detach().float().cpu().double().numpy()


def test_recall_coclustering_vs_kmeans(pb):
    H, kq, kk, iters = 4, 32, 64, 2
    w = video_qkv(4, 32, 32, H, 128, seed=17)          # N = 4096, 64 planted regions per head
    N = w.q.shape[2]
    q, k = w.q.cuda(), w.k.cuda()
    parts = {"coclustering": pb.coclust_assign(q, k, kq, kk, iters, seed=0),
             "kmeans": pb.coclust_assign(q, k, kq, kk, iters, seed=0, kmeans=True)}
    torch.cuda.synchronize()
    fracs = [0.02, 0.05, 0.1, 0.2]
    rows = []
    for h in range(H):
        Q, K = f64(w.q[0, h]), f64(w.k[0, h])
        S = Q @ K.T / math.sqrt(Q.shape[1])
        A = np.exp(S - S.max(1, keepdims=True))
        A /= A.sum(1, keepdims=True)
        ref = svoo.reference_pairs(A, 0.5)
        row = {"head": h, "ref_pairs": int(ref.sum())}
        for name, st in parts.items():
            cnt = svoo.block_pair_counts(ref, st["lq"][0, h].cpu().numpy(), st["lk"][0, h].cpu().numpy(), kq, kk)
            rec = [svoo.block_pair_recall(cnt, max(1, int(f * kq * kk))) for f in fracs]
            assert all(0.0 <= r <= 1.0 for r in rec) and all(a <= b + 1e-12 for a, b in zip(rec, rec[1:]))
            row[name] = {"recall_at_budget_frac": dict(zip(map(str, fracs), rec)),
                         "pairs_to_cover_all": svoo.pairs_to_cover(cnt),
                         "pairs_to_cover_90pct": svoo.pairs_to_cover(cnt, 0.9)}
        rows.append(row)
    mean = {name: {str(f): float(np.mean([r[name]["recall_at_budget_frac"][str(f)] for r in rows])) for f in fracs}
            for name in parts}
    out = {"workload": f"video_qkv 4x32x32 (N={N}), {H} heads, d=128, 64 planted regions, K_q/K_k={kq}/{kk}, "
                       f"{iters} iterations", "reference": "top-50% attention mass token pairs (P:182)",
           "budget": "block pairs = frac x K_q x K_k, each method its best pairs (P:183, R19)",
           "mean_recall": mean, "per_head": rows}
    path = os.environ.get("RECALL_OUT")
    if path:
        with open(path, "w") as f:
            json.dump(out, f, indent=1)
    print(json.dumps(mean))
