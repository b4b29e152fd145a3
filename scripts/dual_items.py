"""Cost model (oracle kept sets, one Wan2.1-14B head at a time) of pairing split-KV single-tile items of two
query clusters into one two-Q-tile item over the union of their kept sets (per-set column masks):
greedy pairing by cycles saved, with the measured per-KV-tile costs (pair item 2,735, split item 2,102)."""
import numpy as np, torch, sys, time
sys.path.insert(0, '.')
from oracle import svoo
from synthetic import video_qkv
w = video_qkv(21, 45, 80, 2, 128, seed=0)
for h in range(2):
    f = lambda t: t[0, h].float().double().numpy()
    Q, K = f(w.q), f(w.k)
    r = svoo.cocluster(Q, K, 100, 500, 2, seed=0, h=h, H=40)
    sq = np.bincount(r.Lq, minlength=100); sk = np.bincount(r.Lk, minlength=500)
    sel = svoo.select_blocks(r.Cq, r.Ck, sq, sk, 0.2, 0.95, 0.1, svoo.RULE_FIXED)
    kept = [set(np.asarray(sel.kept[a]).tolist()) for a in range(100)]
    rows = lambda S: sum(sk[c] for c in S)
    tiles = lambda S: -(-rows(S) // 128)
    T = [-(-int(sq[a]) // 128) for a in range(100)]
    singles = [a for a in range(100) if T[a] % 2 == 1 and sq[a] > 0]
    PAIR, SPLIT = 2735, 2102
    cost_split = sum(tiles(kept[a]) * SPLIT for a in singles)
    # greedy: pair singles with the smallest union
    cand = []
    for i, a in enumerate(singles):
        for b in singles[i+1:]:
            u = tiles(kept[a] | kept[b])
            gain = (tiles(kept[a]) + tiles(kept[b])) * SPLIT - u * PAIR
            cand.append((gain, a, b, u))
    cand.sort(reverse=True)
    used = set(); saved = 0; npairs = 0
    for g, a, b, u in cand:
        if g <= 0: break
        if a in used or b in used: continue
        used.add(a); used.add(b); saved += g; npairs += 1
    total = sum((T[a] // 2) * tiles(kept[a]) * PAIR + (T[a] % 2) * tiles(kept[a]) * SPLIT for a in range(100))
    ov = [len(kept[a] & kept[b]) / 100 for a, b in [(c[1], c[2]) for c in cand[:20]]]
    print(f"head {h}: singles {len(singles)}, split cost share {cost_split/total:.3f}, dual pairs {npairs}, saved {saved/total:.4f} of the head's attention cycles; top-20 overlaps {np.round(ov,2)}")
