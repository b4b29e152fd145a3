"""Cost model (float64 oracle kept sets of two synthetic Wan2.1-14B 720p heads, FIXED rho = 0.2) of
row-merging the split-KV single-tile items of two query clusters into ONE 128-row Q tile when their
tail rows fit (rows_a + rows_b <= 128), run over the union of their kept sets with per-row masks, at
the measured per-KV-tile costs (pair item 2,735, split item 2,102 cycles).  Greedy by cycles saved;
mask overhead not included.

    python scripts/tail_merge.py <kq> <kk>
"""
import numpy as np, sys
sys.path.insert(0, '.')
from oracle import svoo
from synthetic import video_qkv
kq, kk = int(sys.argv[1]), int(sys.argv[2])
w = video_qkv(21, 45, 80, 2, 128, seed=0)
PAIR, SPLIT = 2735, 2102
for h in range(2):
    f = lambda t: t[0, h].float().double().numpy()
    Q, K = f(w.q), f(w.k)
    r = svoo.cocluster(Q, K, kq, kk, 2, seed=0, h=h, H=40)
    sq = np.bincount(r.Lq, minlength=kq); sk = np.bincount(r.Lk, minlength=kk)
    sel = svoo.select_blocks(r.Cq, r.Ck, sq, sk, 0.2, 0.95, 0.1, svoo.RULE_FIXED)
    kept = [set(np.asarray(sel.kept[a]).tolist()) for a in range(kq)]
    rows = lambda S: sum(sk[c] for c in S)
    tiles = lambda S: -(-rows(S) // 128)
    T = [-(-int(sq[a]) // 128) for a in range(kq)]
    tail = [int(sq[a]) - 128 * (T[a] - 1) for a in range(kq)]
    singles = [a for a in range(kq) if T[a] % 2 == 1 and sq[a] > 0]
    total = sum((T[a] // 2) * tiles(kept[a]) * PAIR + (T[a] % 2) * tiles(kept[a]) * SPLIT for a in range(kq))
    cost_split = sum(tiles(kept[a]) * SPLIT for a in singles)
    # (B) row-merge: two single tails with rows_a + rows_b <= 128 -> one tile over the union (SPLIT cost)
    cand = []
    for i, a in enumerate(singles):
        for b in singles[i + 1:]:
            if tail[a] + tail[b] > 128: continue
            u = tiles(kept[a] | kept[b])
            gain = (tiles(kept[a]) + tiles(kept[b]) - u) * SPLIT
            cand.append((gain, a, b))
    cand.sort(reverse=True)
    used = set(); saved = 0; n = 0
    for g, a, b in cand:
        if g <= 0: break
        if a in used or b in used: continue
        used.add(a); used.add(b); saved += g; n += 1
    print(f"{kq}/{kk} head {h}: singles {len(singles)} (tail rows mean {np.mean([tail[a] for a in singles]):.0f}), "
          f"split share {cost_split/total:.3f}, row-merged pairs {n}, saved {saved/total:.4f} of attention cycles", flush=True)
