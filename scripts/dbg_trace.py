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
names = ['P:K issued', 'P:V issued', 'M:k_full', 'M:v_full', 'M:p0', 'S0:s_full', 'S0:p_arr', 'S1:s_full', 'S1:p_arr', '-', '-', 'M:p1']
nt = int((buf[5] > 0).sum())
t0 = buf[buf > 0].min()
print('rc', rc, 'tiles', nt, 'tile1 active', (buf[7] > 0).any())
for j in list(range(0, 6)) + list(range(nt // 2, nt // 2 + 4)):
    print(j, ' '.join(f"{names[e]}={(buf[e, j] - t0) if buf[e, j] else -1:>8}" for e in (0, 1, 2, 3, 4, 11, 5, 6, 7, 8)))
d = lambda a, b: np.diff(buf[a, :nt]) if b is None else (buf[b, :nt] - buf[a, :nt])
print('period S0 (s_full->s_full) median', np.median(np.diff(buf[5, 1:nt])))
print('softmax0 (s_full->p_arr) median', np.median(buf[6, 1:nt] - buf[5, 1:nt]))
print('p_arr0 -> M:p0 seen median', np.median(buf[4, 1:nt] - buf[6, 1:nt]))
print('M:p0 -> M:v_full median', np.median(buf[3, 1:nt] - buf[4, 1:nt]))
print('M:p0(j) -> S0:s_full(j+1) median', np.median(buf[5, 2:nt] - buf[4, 1:nt - 1]))
print('V issued(j) -> M:v_full(j) median', np.median(buf[3, 1:nt] - buf[1, 1:nt]))
print('K issued(j) -> M:k_full(j) median', np.median(buf[2, 2:nt] - buf[0, 2:nt]))

print('K: k_empty wait done -> issued', np.median(buf[0, 2:nt] - buf[9, 2:nt]), ' prev V issued -> k_empty done', np.median(buf[9, 2:nt] - buf[1, 1:nt-1]))
print('V: v_empty wait done -> issued', np.median(buf[1, 2:nt] - buf[10, 2:nt]), ' K issued -> v_empty done', np.median(buf[10, 2:nt] - buf[0, 3:nt+1]))
print('softmax0: s_full->masked', np.median(buf[16, 1:nt] - buf[5, 1:nt]), 'masked->max', np.median(buf[12, 1:nt] - buf[16, 1:nt]))
print('softmax0: s_full->max', np.median(buf[12, 1:nt] - buf[5, 1:nt]), 'max->exp done', np.median(buf[14, 1:nt] - buf[12, 1:nt]), 'exp done->arrive', np.median(buf[6, 1:nt] - buf[14, 1:nt]))
