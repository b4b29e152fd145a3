"""Parity at the paper's own operating point on the Wan2.1-14B 720p head shape (N = 75,600, d = 128):
K_q = 256 query / K_k = 1024 key clusters, the DENSITY rule with tau = 0.95, theta = 0.1
 and a per-head budget of a synthetic offline profile, through
the fused layer entry.  Four heads (the layer's launch shape at H = 4), stage by stage against the
oracle fed the GPU's own upstream state, with the SURVEY §8c tolerances — the configuration the
bench's 256/1024 sweep cells time, which the 100/500 full-size tests do not cover (CTA-pair
assignment with 4 N-chunks, 74-row key clusters, mostly single-tile split-KV attention items)."""
import math

import numpy as np
import pytest
import torch

from oracle import svoo

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

KQ, KK, IT, H = 256, 1024, 2, 4


@pytest.fixture(scope="module")
def run():
    import paper_2603_18636_b200 as pb
    from synthetic import config_workload
    w = config_workload("wan14b_720p", device="cuda", H=H)
    budget = torch.tensor([0.12, 0.3, 0.05, 0.9], device="cuda")  # includes the DENSITY max branch (1 - b <= theta)
    st = pb.coclust_assign(w.q, w.k, KQ, KK, IT, seed=3)
    n_keep, kept = pb.block_select(st["cq"], st["ck"], st["offs_q"], st["offs_k"], budget, 0.95, 0.1,
                                   pb.RULE_DENSITY)
    o = pb.coclust_sparse_attention(w.q, w.k, w.v, KQ, KK, IT, budget, rule=pb.RULE_DENSITY, seed=3)
    torch.cuda.synchronize()
    return dict(pb=pb, w=w, st=st, n_keep=n_keep, kept=kept, o=o, budget=budget.cpu().numpy())


def f64(t):
    return t.detach().float().cpu().double().numpy()


def test_paper_defaults_first_halfstep_labels(run):
    pb, w = run["pb"], run["w"]
    N = w.q.shape[2]
    for h in range(H):
        iq = svoo.sample_anchor_indices(N, KQ, 3, 0, h, H, 0)
        ik = svoo.sample_anchor_indices(N, KK, 3, 0, h, H, 1)
        Q, K = f64(w.q[0, h]), f64(w.k[0, h])
        ca, cs = Q[iq], K[ik]
        lab = pb.coclust_assign_step(w.k[:, h:h + 1].contiguous(), torch.from_numpy(ca).float()[None, None].cuda(),
                                     torch.from_numpy(cs).float()[None, None].cuda())[0, 0].cpu().numpy()
        res = svoo.assign_step(K, ca, cs)
        ok = res.gap >= 1e-4
        assert np.sum((lab != res.labels) & ok) == 0, h
        assert ok.mean() > 0.97


def test_paper_defaults_permutation_and_centroids(run):
    st, w = run["st"], run["w"]
    for h in range(H):
        for side, X, k in (("q", w.q, KQ), ("k", w.k, KK)):
            lab = st["l" + side][0, h].cpu().numpy()
            perm, offs = svoo.counting_sort(lab, k)
            assert np.array_equal(st["perm_" + side][0, h].cpu().numpy(), perm)
            assert np.array_equal(st["offs_" + side][0, h].cpu().numpy(), offs)
            C = st["c" + side][0, h].cpu().double().numpy()
            Xh = f64(X[0, h])
            sizes = np.bincount(lab, minlength=k)
            sums = np.zeros((k, Xh.shape[1]))
            np.add.at(sums, lab, Xh)
            ne = sizes > 0
            np.testing.assert_allclose(C[ne], sums[ne] / sizes[ne, None], rtol=1e-5, atol=1e-6)


def test_paper_defaults_density_selection_bitexact(run):
    st = run["st"]
    checked = 0
    for h in range(H):
        Cq = st["cq"][0, h].cpu().double().numpy()
        Ck = st["ck"][0, h].cpu().double().numpy()
        sq = np.diff(st["offs_q"][0, h].cpu().numpy())
        sk = np.diff(st["offs_k"][0, h].cpu().numpy())
        A = Cq @ Ck.T
        clean = all(np.min(np.abs(np.diff(np.sort(A[a, sk > 0])[::-1])) /
                           np.maximum(np.abs(np.sort(A[a, sk > 0])[::-1][:-1]), 1e-300)) >= 1e-9
                    for a in range(KQ) if sq[a] > 0)
        if not clean:
            continue
        ref = svoo.select_blocks(Cq, Ck, sq, sk, float(np.float32(run["budget"][h])), 0.95, 0.1, svoo.RULE_DENSITY,
                                 d_head=128)
        n = int(run["n_keep"][0, h])
        assert n == ref.n_keep, h
        assert np.array_equal(run["kept"][0, h, :, :n].cpu().numpy(), ref.kept), h
        checked += 1
    assert checked >= 2, f"only {checked} margin-clean heads"


def test_paper_defaults_attention_sampled_rows(run):
    st, w, o = run["st"], run["w"], run["o"]
    rng = np.random.default_rng(1)
    for h in range(H):
        Lq = st["lq"][0, h].cpu().numpy()
        Lk = st["lk"][0, h].cpu().numpy()
        n = int(run["n_keep"][0, h])
        kept = run["kept"][0, h, :, :n].cpu().numpy()
        Q, K, V = f64(w.q[0, h]), f64(w.k[0, h]), f64(w.v[0, h])
        rows = rng.choice(Q.shape[0], 256, replace=False)
        ref = []
        for i in rows:
            allowed = np.nonzero(np.isin(Lk, kept[Lq[i]]))[0]
            s = (K[allowed] @ Q[i]) / math.sqrt(Q.shape[1])
            e = np.exp(s - s.max())
            ref.append((e @ V[allowed]) / e.sum())
        err = np.abs(f64(o[0, h])[rows] - np.stack(ref))
        assert err.max() <= 2e-2 and err.mean() <= 5e-3, (h, err.max(), err.mean())
