import numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_2603_18636_b200 as pb
from oracle import svoo
from synthetic import random_qkv
d, N = 128, 256
w = random_qkv(1, 1, N, d, seed=5)
Lq = np.arange(N) % 4; Lk = np.arange(N)
pq, oq = svoo.counting_sort(Lq, 4); pk, ok = svoo.counting_sort(Lk, N)
kept = np.full((4, N), -1, np.int64); kept[:, 0] = [3, 77, 150, 255]
t = lambda a: torch.from_numpy(np.asarray(a).astype(np.int32))[None, None].cuda()
O = pb.block_sparse_attn(w.q.cuda(), w.k.cuda(), w.v.cuda(), t(pq), t(oq), t(pk), t(ok),
                         torch.ones(1, 1, dtype=torch.int32).cuda(), t(kept))
exp = w.v[0, 0][torch.tensor([3, 77, 150, 255])[Lq]]
O = O[0, 0].cpu().float(); e = exp.float()
rel = (O / e)
bad = (O != e)
print("mismatching elements", int(bad.sum()), "rows", torch.nonzero(bad.any(1)).flatten().tolist()[:20])
r = (O[bad] / e[bad])
print("ratio O/exp over mismatches: min %.6f max %.6f" % (r.min(), r.max()) if bad.any() else "exact")
# logits of the kept key for rows: q.k*scale*log2e
q = w.q[0, 0].float(); k = w.k[0, 0].float()
s = (q * k[torch.tensor([3, 77, 150, 255])[Lq]]).sum(1) * d ** -0.5 * 1.4426950408889634
print("scaled logits of bad rows", s[bad.any(1)][:8].tolist())
import os
if 'dbg' in os.environ.get('COCLUST_LIB', ''):
    raw = pb.block_sparse_attn(w.q.cuda(), w.k.cuda(), w.v.cuda(), t(pq), t(oq), t(pk), t(ok),
                               torch.ones(1, 1, dtype=torch.int32).cuda(), t(kept))[0, 0].cpu()
    u32 = raw.view(torch.int32)[:, :8]
    f = u32.view(torch.float32)
    for i in [0, 1, 5, 17, 48]:
        print(i, "m=%.6f l=%.6f s0=%.6f s1=%.6g mw0=%08x nt=%d U=%d n=%d" % (f[i,0], f[i,1], f[i,2], f[i,3], u32[i,4] & 0xffffffff, u32[i,5], u32[i,6], u32[i,7]),
              "expected s*sl=%.6f" % float(s[i]))
