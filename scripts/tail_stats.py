"""Q-tile padding statistics of one layer (bench workload): how much of the attention work is the
partial last Q tile of each cluster, and what merging two clusters' tails into one 128-row tile
(KV stream = union of their kept key clusters) would save.  Measurement only, not product code.

  python scripts/tail_stats.py [--config wan14b_720p] [--budget 0.2]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_18636_b200 as pb  # noqa: E402
from synthetic import CONFIGS, video_qkv  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="wan14b_720p")
ap.add_argument("--kq", type=int, default=100)
ap.add_argument("--kk", type=int, default=500)
ap.add_argument("--budget", type=float, default=0.2)
ap.add_argument("--heads", type=int, default=40)
a = ap.parse_args()
c = CONFIGS[a.config]
dev = torch.device("cuda")
full = video_qkv(c["T"], c["Hs"], c["Ws"], c["H"], c["d"], seed=0, device=dev)
H = min(a.heads, c["H"])
q, k = full.q[:, :H].contiguous(), full.k[:, :H].contiguous()
st = pb.coclust_assign(q, k, a.kq, a.kk, 2, seed=0, head_offset=0, heads_total=c["H"])
budget = torch.full((H,), a.budget, dtype=torch.float32, device=dev)
n_keep, kept = pb.block_select(st["cq"], st["ck"], st["offs_q"], st["offs_k"], budget, rule=pb.RULE_FIXED)
offs_q, offs_k = st["offs_q"].cpu().numpy()[0], st["offs_k"].cpu().numpy()[0]
n_keep, kept = n_keep.cpu().numpy()[0], kept.cpu().numpy()[0]

tot_issued = tot_kept = tot_tail = 0.0
save_rand = save_greedy = 0.0
for h in range(H):
    qs = np.diff(offs_q[h])
    ks = np.diff(offs_k[h])
    sets, keys = [], []
    for a_ in range(a.kq):
        s = kept[h, a_, :n_keep[h]]
        sets.append(set(s.tolist()))
        keys.append(int(ks[s].sum()))
    keys = np.array(keys, dtype=np.float64)
    kt = np.ceil(keys / 128) * 128
    tiles = np.ceil(qs / 128)
    tot_issued += float((tiles * 128 * kt).sum())
    tot_kept += float((qs * keys).sum())
    tail = qs % 128
    has = (tail > 0) & (qs > 0)
    tot_tail += float((has * 128 * kt).sum())
    idx = [i for i in range(a.kq) if has[i]]
    # greedy: largest tail first, partner = fitting tail with the largest kept-set overlap
    free = set(idx)
    for i in sorted(idx, key=lambda i: -tail[i]):
        if i not in free:
            continue
        free.discard(i)
        best, bj = 0.0, None
        for j in free:
            if tail[i] + tail[j] <= 128:
                u = len(sets[i] | sets[j])
                un = float(sum(ks[list(sets[i] | sets[j])]))
                sv = kt[i] + kt[j] - np.ceil(un / 128) * 128
                if sv > best:
                    best, bj = sv, j
        if bj is not None:
            free.discard(bj)
            save_greedy += 128 * best
    # random-order pairing (first fitting partner)
    free = list(idx)
    rng = np.random.default_rng(h)
    rng.shuffle(free)
    used = set()
    for i in free:
        if i in used:
            continue
        used.add(i)
        for j in free:
            if j not in used and tail[i] + tail[j] <= 128:
                used.add(j)
                un = float(sum(ks[list(sets[i] | sets[j])]))
                save_rand += 128 * (kt[i] + kt[j] - np.ceil(un / 128) * 128)
                break
res = dict(config=a.config, heads=H, kq=a.kq, kk=a.kk, budget=a.budget,
           padding_frac=1 - tot_kept / tot_issued, tail_work_frac=tot_tail / tot_issued,
           merge_saving_greedy_frac=save_greedy / tot_issued, merge_saving_random_frac=save_rand / tot_issued)
print(json.dumps(res))
