"""Per-event clock64 trace of one attention CTA (debug variant lib, -DCS_ATTN_DEBUG)."""
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
L.cs_debug_attn_trace.restype = ctypes.c_int
rc = L.cs_debug_attn_trace(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes))
nt = int((buf[5] > 0).sum())
print('rc', rc, 'tiles', nt, 'tile1 active', (buf[7] > 0).any())
med = lambda x: float(np.median(x))
s = slice(2, nt - 2)
sn = slice(3, nt - 1)
print('period S0 (s_full->s_full)', med(buf[5, sn] - buf[5, s]))
print('softmax0 s_full->p_arr', med(buf[6, s] - buf[5, s]), '| s_full->masked', med(buf[16, s] - buf[5, s]),
      'masked->max', med(buf[12, s] - buf[16, s]), 'max->exp done', med(buf[14, s] - buf[12, s]), 'exp->arr', med(buf[6, s] - buf[14, s]))
print('softmax0 idle: p_arr(j) -> s_full(j+1)', med(buf[5, sn] - buf[6, s]))
print('MMA: p_arr0(j) -> PV0 issued', med(buf[4, s] - buf[6, s]), '| QK(j+1) k_full seen -> s_full0(j+1)', med(buf[5, sn] - buf[2, sn]))
print('MMA: v_full seen(j) - p0 seen(j)', med(buf[3, s] - buf[4, s]))
print('producer: K issue after k_empty', med(buf[0, s] - buf[9, s]), 'V issue after v_empty', med(buf[1, s] - buf[10, s]))
print('K issued(j) -> k_full seen(j)', med(buf[2, s] - buf[0, s]), 'V issued(j) -> v_full seen(j)', med(buf[3, s] - buf[1, s]))
j = np.arange(3, nt - 3)
print('MMA: QK(j+1) issue time [k_full(j+1) seen -> v_full(j) seen]', med(buf[3, j] - buf[2, j + 1]))
print('MMA: prev PV1(j-1) issued -> k_full(j+1) seen', med(buf[2, j + 1] - buf[11, j - 1]))
print('MMA: v_full(j) seen -> p0(j) seen', med(buf[4, j] - buf[3, j]), ' p0 -> p1 seen', med(buf[11, j] - buf[4, j]))
print('producer K: issued(j+1) vs MMA k_full(j+1) seen', med(buf[2, j + 1] - buf[0, j + 1]))
print('raw j=10..13 events (rel):')
for jj in range(10, 14):
    t0 = buf[5, jj]
    print(jj, {n: int(buf[e, jj] - t0) for n, e in [('Kiss', 0), ('Viss', 1), ('kf', 2), ('vf', 3), ('p0', 4), ('p1', 11), ('S0', 5), ('P0', 6), ('S1', 7), ('P1', 8)]})
