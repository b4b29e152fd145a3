"""Per-event clock64 trace of one attention CTA (v3 layout: 128-key tiles, S/P aliasing)."""
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
print('tiles', nt, 'period', med(buf[5, sn] - buf[5, s]))
print('softmax0', med(buf[6, s] - buf[5, s]), '| ld->masked', med(buf[16, s] - buf[5, s]), 'max', med(buf[12, s] - buf[16, s]),
      'exp', med(buf[14, s] - buf[12, s]), 'st+arrive', med(buf[6, s] - buf[14, s]))
print('p_arr0 -> MMA sees p0', med(buf[4, s] - buf[6, s]), '| MMA p0 seen -> s_full0(j+1)', med(buf[5, sn] - buf[4, s]))
print('S1 start - S0 start', med(buf[7, s] - buf[5, s]))
