"""Per-CTA timeline of the attention kernel (debug variant, %globaltimer): setup time, time to the
first S tile, loop time, and the gap between consecutive CTAs on the same SM."""
import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, '.')
import paper_2603_18636_b200 as pb
from synthetic import video_qkv
H = int(os.environ.get('H', '8'))
w = video_qkv(21, 45, 80, H, 128, seed=0, device='cuda')
budget = torch.full((H,), 0.2, device='cuda')
for _ in range(2):
    o = pb.coclust_sparse_attention(w.q, w.k, w.v, 100, 500, 2, budget, rule=pb.RULE_FIXED)
torch.cuda.synchronize()
buf = np.zeros((65536, 8), np.int64)
pb.lib().cs_debug_attn_cta(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes))
v = buf[buf[:, 3] > 0]
t0 = v[:, 0].min()
print("ctas", len(v), "kernel span us %.1f" % ((v[:, 3].max() - t0) / 1e3))
dur = (v[:, 3] - v[:, 0]) / 1e3
setup = (v[:, 1] - v[:, 0]) / 1e3
first = (v[:, 2] - v[:, 1]) / 1e3
print("CTA duration us: median %.1f  mean %.1f" % (np.median(dur), dur.mean()))
print("setup (entry -> tables/TMEM ready) us: median %.2f mean %.2f" % (np.median(setup), setup.mean()))
print("ready -> first S tile us: median %.2f mean %.2f" % (np.median(first), first.mean()))
ghz = (v[:, 7] - v[:, 6]) / (v[:, 3] - v[:, 0])
print("effective SM clock GHz (clock64 / globaltimer over each CTA): median %.3f  p10 %.3f  p90 %.3f" %
      (np.median(ghz), np.percentile(ghz, 10), np.percentile(ghz, 90)))
nt = v[:, 5] & 0xfffff
sp = (v[:, 5] >> 20) & 1
loop = dur - setup - first
print("per-KV-tile loop us: median %.3f" % np.median(loop / np.maximum(nt, 1)))
for flag, name in ((0, "pair items"), (1, "split-KV single-tile items")):
    m = sp == flag
    if m.any():
        print(f"{name}: {m.sum()} CTAs, per-KV-tile us median %.3f (cycles %.0f), duration median %.1f" %
              (np.median(loop[m] / np.maximum(nt[m], 1)), np.median(loop[m] * 1e3 * ghz[m] / np.maximum(nt[m], 1)),
               np.median(dur[m])))
gaps = []
for sm in np.unique(v[:, 4]):
    x = v[v[:, 4] == sm]
    x = x[np.argsort(x[:, 0])]
    gaps.extend(((x[1:, 0] - x[:-1, 3]) / 1e3).tolist())
print("gap between CTAs on one SM us: median %.2f mean %.2f" % (np.median(gaps), np.mean(gaps)))
print("overhead share (setup + first S + gap) / duration: %.3f" % ((np.median(setup) + np.median(first) + np.median(gaps)) / np.median(dur)))
