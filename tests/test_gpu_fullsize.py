"""Parity at BASELINE.json's full sizes (Wan2.1-14B 720p: N=75,600, H=40; HunyuanVideo 720p:
N=118,800, H=24; Wan2.1-1.3B 480p: N=32,760, H=12; d=128, 100/500 clusters, I_max=2, FIXED
rho=0.2) in the launch configuration bench.py times.  The oracle cannot run the
whole layer in seconds, so each stage is checked on sampled heads / rows against the oracle fed
the GPU's own upstream state (teacher forcing), with the SURVEY §8c tolerances."""
import math

import numpy as np
import pytest
import torch

from oracle import svoo

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

KQ, KK, IT, BUDGET = 100, 500, 2, 0.2


@pytest.fixture(scope="module", params=["wan14b_720p", "hunyuan_720p", "wan1.3b_480p"])
def run(request):
    import paper_2603_18636_b200 as pb
    from synthetic import config_workload
    w = config_workload(request.param, device="cuda")
    H = w.q.shape[1]
    budget = torch.full((H,), BUDGET, device="cuda")
    st = pb.coclust_assign(w.q, w.k, KQ, KK, IT, seed=0)
    n_keep, kept = pb.block_select(st["cq"], st["ck"], st["offs_q"], st["offs_k"], budget, 0.95, 0.1,
                                   pb.RULE_FIXED)
    o = pb.coclust_sparse_attention(w.q, w.k, w.v, KQ, KK, IT, budget, rule=pb.RULE_FIXED, seed=0)
    torch.cuda.synchronize()
    return dict(pb=pb, w=w, st=st, n_keep=n_keep, kept=kept, o=o, H=H, heads=(0, H // 2, H - 1), name=request.param)


def f64(t):
    return t.detach().float().cpu().double().numpy()


def test_fullsize_first_halfstep_labels(run):
    """Step A of iteration 1 from the R4 initial centroids: GPU labels == oracle labels except
    near-ties (gap < 1e-4)."""
    pb, w = run["pb"], run["w"]
    N = w.q.shape[2]
    for h in run["heads"]:
        iq = svoo.sample_anchor_indices(N, KQ, 0, 0, h, run["H"], 0)
        ik = svoo.sample_anchor_indices(N, KK, 0, 0, h, run["H"], 1)
        K = f64(w.k[0, h])
        Q = f64(w.q[0, h])
        ca, cs = Q[iq], K[ik]
        lab = pb.coclust_assign_step(w.k[:, h:h + 1].contiguous(),
                                     torch.from_numpy(ca).float()[None, None].cuda(),
                                     torch.from_numpy(cs).float()[None, None].cuda())[0, 0].cpu().numpy()
        res = svoo.assign_step(K, ca, cs)
        ok = res.gap >= 1e-4
        assert np.sum((lab != res.labels) & ok) == 0
        assert ok.mean() > 0.98


def test_fullsize_permutation_bitexact(run):
    st = run["st"]
    for h in run["heads"]:
        for side, k in (("q", KQ), ("k", KK)):
            lab = st["l" + side][0, h].cpu().numpy()
            perm, offs = svoo.counting_sort(lab, k)
            assert np.array_equal(st["perm_" + side][0, h].cpu().numpy(), perm)
            assert np.array_equal(st["offs_" + side][0, h].cpu().numpy(), offs)


def test_fullsize_centroids_are_member_means(run):
    st, w = run["st"], run["w"]
    for h in run["heads"][:2]:
        for side, X, k in (("q", w.q, KQ), ("k", w.k, KK)):
            lab = st["l" + side][0, h].cpu().numpy()
            C = st["c" + side][0, h].cpu().double().numpy()
            Xh = f64(X[0, h])
            sizes = np.bincount(lab, minlength=k)
            sums = np.zeros((k, Xh.shape[1]))
            np.add.at(sums, lab, Xh)
            ne = sizes > 0
            np.testing.assert_allclose(C[ne], sums[ne] / sizes[ne, None], rtol=1e-5, atol=1e-6)


def test_fullsize_selection_bitexact(run):
    st = run["st"]
    checked = 0
    for h in range(run["H"]):
        Cq = st["cq"][0, h].cpu().double().numpy()
        Ck = st["ck"][0, h].cpu().double().numpy()
        sq = np.diff(st["offs_q"][0, h].cpu().numpy())
        sk = np.diff(st["offs_k"][0, h].cpu().numpy())
        A = Cq @ Ck.T
        # margin check: adjacent sorted Abar values must be separated
        ok = True
        for a in range(KQ):
            v = np.sort(A[a, sk > 0])[::-1]
            if np.min(np.abs(np.diff(v)) / np.maximum(np.abs(v[:-1]), 1e-300)) < 1e-9:
                ok = False
                break
        if not ok:
            continue
        ref = svoo.select_blocks(Cq, Ck, sq, sk, BUDGET, 0.95, 0.1, svoo.RULE_FIXED, d_head=128)
        n = int(run["n_keep"][0, h])
        assert n == ref.n_keep
        assert np.array_equal(run["kept"][0, h, :, :n].cpu().numpy(), ref.kept)
        checked += 1
        if checked == 6:
            break
    assert checked >= 4, f"only {checked} margin-clean heads"


def test_fullsize_attention_sampled_rows(run):
    st, w, o = run["st"], run["w"], run["o"]
    rng = np.random.default_rng(0)
    for h in run["heads"]:
        Lq = st["lq"][0, h].cpu().numpy()
        Lk = st["lk"][0, h].cpu().numpy()
        n = int(run["n_keep"][0, h])
        kept = run["kept"][0, h, :, :n].cpu().numpy()
        Q, K, V = f64(w.q[0, h]), f64(w.k[0, h]), f64(w.v[0, h])
        rows = rng.choice(Q.shape[0], 384, replace=False)
        ref = np.stack([_row(Q, K, V, Lq, Lk, kept, i) for i in rows])
        got = f64(o[0, h])[rows]
        err = np.abs(got - ref)
        assert err.max() <= 2e-2 and err.mean() <= 5e-3, (err.max(), err.mean())


def _row(Q, K, V, Lq, Lk, kept, i):
    allowed = np.nonzero(np.isin(Lk, kept[Lq[i]]))[0]
    s = (K[allowed] @ Q[i]) / math.sqrt(Q.shape[1])
    e = np.exp(s - s.max())
    return (e @ V[allowed]) / e.sum()


def test_fullsize_teacher_forced_all_halfsteps(run):
    """SURVEY §8c P1 chained through ALL 2 * I_max half-steps of Alg. 1 at full size: the oracle
    runs Alg. 1 on the head (seed 0, global head h), and each GPU half-step fed the oracle's
    (C_anchor, C_self) of that half-step — Step A of iterations 1 and 2 on C_q^(i-1) / C_k^(i-1),
    Step B on the NEW C_k^(i) and the old C_q^(i-1) — gives the oracle's labels
    except near-ties (gap < 1e-4).  Given the oracle's labels, the GPU centroid update (P2) is
    within 1e-5 of the oracle's C^(i).  Three heads of Wan2.1-14B 720p, one of the others."""
    pb, w = run["pb"], run["w"]
    heads = run["heads"] if run["name"] == "wan14b_720p" else run["heads"][:1]
    for h in heads:
        Q, K = f64(w.q[0, h]), f64(w.k[0, h])
        cc = svoo.cocluster(Q, K, KQ, KK, IT, seed=0, h=h, H=run["H"])
        assert [t["side"] for t in cc.trace] == ["k", "q", "k", "q"]
        for t in cc.trace:
            X = w.k if t["side"] == "k" else w.q
            xh = X[:, h:h + 1].contiguous()
            ca = torch.from_numpy(t["C_anchor"]).float()[None, None].cuda()
            cs = torch.from_numpy(t["C_self"]).float()[None, None].cuda()
            lab = pb.coclust_assign_step(xh, ca, cs)[0, 0].cpu().numpy()
            ok = t["gap"] >= 1e-4
            assert np.sum((lab != t["labels"]) & ok) == 0, (h, t["it"], t["side"])
            assert ok.mean() > 0.98
            k = t["C_self"].shape[0]
            perm, offs = pb.coclust_permute(torch.from_numpy(t["labels"].astype(np.int32))[None].cuda(), k)
            c = cs.clone()
            pb.coclust_update_centroids(xh, perm[None], offs[None], c)
            torch.cuda.synchronize()
            got = c[0, 0].double().cpu().numpy()
            ne = np.bincount(t["labels"], minlength=k) > 0
            np.testing.assert_allclose(got[ne], t["C_new"][ne], rtol=1e-5, atol=1e-5)
            np.testing.assert_array_equal(got[~ne], t["C_self"][~ne].astype(np.float32))


def test_fullsize_attention_every_row_of_one_head(run):
    """P5 on every one of the N rows of head 0 (75,600 at Wan2.1-14B 720p), element by element,
    against the oracle's masked softmax on the GPU's partition and kept blocks."""
    st, w, o = run["st"], run["w"], run["o"]
    h = 0
    Lq = st["lq"][0, h].cpu().numpy()
    Lk = st["lk"][0, h].cpu().numpy()
    n = int(run["n_keep"][0, h])
    kept = run["kept"][0, h, :, :n].cpu().numpy()
    ref = svoo.sparse_attention(f64(w.q[0, h]), f64(w.k[0, h]), f64(w.v[0, h]), Lq, Lk, kept)
    err = np.abs(f64(o[0, h]) - ref)
    assert err.shape[0] == w.q.shape[2]
    assert err.max() <= 2e-2 and err.mean() <= 5e-3, (err.max(), err.mean())
