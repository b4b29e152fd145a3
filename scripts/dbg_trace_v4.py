"""Per-event clock64 trace of one attention CTA (128-key tiles, P stored in two halves).
Events: 5/7 S(j) seen by softmax 0/1, 16/17 S loaded+masked, 12/13 row max done, 14/15 first P
half arrived, 6/8 second P half arrived, 3 MMA sees V(j), 4/11 PV0/PV1(j) issued, 2 MMA sees K(j+1)."""
import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, '.')
import paper_2603_18636_b200 as pb
from synthetic import video_qkv
H = int(os.environ.get('H', '4'))
w = video_qkv(21, 45, 80, H, 128, seed=0, device='cuda')
budget = torch.full((H,), 0.2, device='cuda')
for _ in range(2):
    o = pb.coclust_sparse_attention(w.q, w.k, w.v, 100, 500, 2, budget, rule=pb.RULE_FIXED)
torch.cuda.synchronize()
buf = np.zeros((20, 4096), np.int64)
L = pb.lib()
rc = L.cs_debug_attn_trace(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes))
nt = int((buf[5] > 0).sum())
med = lambda x: float(np.median(x))
s, sn = slice(2, nt - 2), slice(3, nt - 1)
print('tiles', nt, 'period S0', med(buf[5, sn] - buf[5, s]), 'period S1', med(buf[7, sn] - buf[7, s]))
for tq, (e_s, e_m, e_x, e_h, e_p) in enumerate([(5, 16, 12, 14, 6), (7, 17, 13, 15, 8)]):
    print(f'softmax{tq}: total', med(buf[e_p, s] - buf[e_s, s]), '| ld+mask', med(buf[e_m, s] - buf[e_s, s]),
          'max', med(buf[e_x, s] - buf[e_m, s]), 'half0 exp+st+arrive', med(buf[e_h, s] - buf[e_x, s]),
          'half1', med(buf[e_p, s] - buf[e_h, s]))
print('PV0 issued after P0 done', med(buf[4, s] - buf[6, s]), '| PV0 issued -> S0(j+1) seen', med(buf[5, sn] - buf[4, s]))
print('PV1 issued after P1 done', med(buf[11, s] - buf[8, s]), '| PV1 issued -> S1(j+1) seen', med(buf[7, sn] - buf[11, s]))
print('S1 start - S0 start', med(buf[7, s] - buf[5, s]), '| S0(j+1) - P1(j) done', med(buf[5, sn] - buf[8, s]))
print('MMA sees V(j) - S0(j) seen', med(buf[3, s] - buf[5, s]), '| MMA sees K(j+1) - S0(j) seen', med(buf[2, s] - buf[5, s]))
print('raw first 6 tiles (rel. to S0(0)):')
t0 = buf[5, 0]
for e in [5, 16, 12, 14, 6, 7, 17, 13, 15, 8, 3, 4, 2, 11]:
    print(e, list(buf[e, :6] - t0))
