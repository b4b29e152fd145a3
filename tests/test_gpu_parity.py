"""GPU parity: every C-ABI entry against the float64 oracle on the same seeded inputs
(SURVEY §8c protocol P1-P6).  Tolerances (BASELINE.json north_star):
  permutation / offsets / block masks: bit-exact given the same labels (P3, P4)
  assignments: identical except tokens whose oracle gap (D2-D1)/D2 < 1e-4 (P1)
  centroids: relative 1e-5 of the fp64 mean (P2)
  attention (bf16 out): max-abs <= 2e-2 and mean-abs <= 5e-3 (P5)
"""
import math

import numpy as np
import pytest
import torch

from oracle import svoo
from synthetic import config_workload, random_labels, random_qkv, video_qkv

pytestmark = pytest.mark.gpu

GAP_TOL = 1e-4
ATOL_MAX, ATOL_MEAN = 2e-2, 5e-3


@pytest.fixture(scope="module")
def pb():
    from paper_2603_18636_b200 import build
    build.build()
    import paper_2603_18636_b200 as m
    m.lib()
    return m


def f64(t):
    return t.detach().float().cpu().double().numpy()


# ------------------------------------------------------------------------- P3 permutation
@pytest.mark.parametrize("BH,N,K", [(3, 5000, 17), (2, 75600, 500), (1, 2048, 16), (2, 777, 1),
                                    (1, 100, 100)])
def test_permute_bitexact(pb, BH, N, K):
    lab = random_labels(BH, N, K, seed=N + K, empty=(0, K // 2) if K > 3 else ())
    perm, offs = pb.coclust_permute(lab.cuda(), K)
    torch.cuda.synchronize()
    for bh in range(BH):
        p_ref, o_ref = svoo.counting_sort(lab[bh].numpy(), K)
        assert np.array_equal(perm[bh].cpu().numpy(), p_ref)
        assert np.array_equal(offs[bh].cpu().numpy(), o_ref)


def test_permute_sorted_labels_and_single_token():
    import paper_2603_18636_b200 as m
    lab = torch.arange(8, dtype=torch.int32).repeat_interleave(3)[None]  # already sorted
    perm, offs = m.coclust_permute(lab.cuda(), 8)
    assert torch.equal(perm.cpu()[0], torch.arange(24, dtype=torch.int32))
    lab1 = torch.zeros(1, 1, dtype=torch.int32)
    perm, offs = m.coclust_permute(lab1.cuda(), 1)
    assert perm.item() == 0 and offs.cpu().tolist() == [[0, 1]]


# ------------------------------------------------------------------------- P2 centroid update
@pytest.mark.parametrize("d,N,K", [(64, 2048, 16), (128, 8192, 100), (128, 20000, 8), (64, 9000, 3)])
def test_update_centroids(pb, d, N, K):
    w = random_qkv(1, 2, N, d, seed=3)
    lab = random_labels(2, N, K, seed=5, empty=(1,))
    prev = torch.randn(1, 2, K, d, generator=torch.Generator().manual_seed(1))
    perm, offs = pb.coclust_permute(lab.cuda(), K)
    c = prev.clone().cuda()
    xp = torch.empty(2, N, d, dtype=torch.bfloat16, device="cuda")
    pb.coclust_update_centroids(w.k.cuda(), perm, offs, c, x_perm=xp)
    torch.cuda.synchronize()
    for h in range(2):
        ref = svoo.update_centroids(f64(w.k[0, h]), lab[h].numpy(), prev[0, h].double().numpy())
        got = c[0, h].cpu().double().numpy()
        assert np.array_equal(got[1], prev[0, h, 1].double().numpy())  # empty keeps previous (R5)
        np.testing.assert_allclose(got, ref, rtol=1e-5, atol=1e-6)
        p_ref, _ = svoo.counting_sort(lab[h].numpy(), K)
        assert torch.equal(xp[h].cpu(), w.k[0, h][torch.from_numpy(p_ref)])


# ------------------------------------------------------------------------- P1 assignment
def _check_labels(got, res, ctx=""):
    ok = res.gap >= GAP_TOL
    mism = (got != res.labels) & ok
    assert mism.sum() == 0, f"{ctx}: {mism.sum()} mismatches outside the near-tie band"
    return int((~ok).sum())


@pytest.mark.parametrize("d,N,ka,ks", [(64, 2048, 16, 16), (128, 8192, 100, 500),
                                       (128, 8192, 500, 100), (128, 3000, 37, 300), (64, 1000, 1, 7),
                                       (128, 4096, 256, 1024),
                                       # CTA-pair kernel shapes: d = 64, one chunk of 160 / 288 columns,
                                       # 2 chunks at N % 256 != 0, 4 chunks of 224
                                       (64, 4096, 50, 500), (64, 2000, 10, 129), (128, 2500, 20, 257),
                                       (128, 1300, 30, 777)])
def test_assign_step(pb, d, N, ka, ks):
    w = video_qkv(4, 16, max(1, N // 64), 2, d, seed=ka + ks)
    N = w.q.shape[2]
    g = torch.Generator().manual_seed(ks)
    ca = torch.randn(1, 2, ka, d, generator=g)
    cs = torch.randn(1, 2, ks, d, generator=g)
    lab = pb.coclust_assign_step(w.k.cuda(), ca.cuda(), cs.cuda())
    torch.cuda.synchronize()
    for h in range(2):
        res = svoo.assign_step(f64(w.k[0, h]), ca[0, h].double().numpy(), cs[0, h].double().numpy())
        _check_labels(lab[0, h].cpu().numpy(), res, f"h={h}")


@pytest.mark.parametrize("kmeans", [False, True])
def test_assign_exact_ties_pick_lowest_index(pb, kmeans):
    """R2 on exact ties: duplicated centroid rows give bit-identical scores, so the argmax epilogue
    must return the lower index — pairs inside one 16-column group, across groups, across 128-column
    chunks and in the ragged last group.  Labels must equal the oracle run on the de-duplicated
    centroid set (mapped back to the lower index) outside its near-tie band."""
    d, N, ka, ks = 128, 4096, 100, 500
    dups = {6: 5, 17: 3, 300: 10, 499: 130}  # higher duplicate -> lower original
    w = video_qkv(4, 16, N // 64, 1, d, seed=77)
    N = w.k.shape[2]
    g = torch.Generator().manual_seed(5)
    ca = torch.randn(1, 1, ka, d, generator=g)
    cs = torch.randn(1, 1, ks, d, generator=g)
    for hi, lo in dups.items():
        cs[0, 0, hi] = cs[0, 0, lo]
    if kmeans:
        lab = pb.kmeans_assign_step(w.k.cuda(), cs.cuda())[0, 0].cpu().numpy()
    else:
        lab = pb.coclust_assign_step(w.k.cuda(), ca.cuda(), cs.cuda())[0, 0].cpu().numpy()
    assert not np.isin(lab, list(dups)).any()
    keep = np.array([j for j in range(ks) if j not in dups])
    X, C = f64(w.k[0, 0]), cs[0, 0].double().numpy()[keep]
    res = svoo.kmeans_step(X, C) if kmeans else svoo.assign_step(X, ca[0, 0].double().numpy(), C)
    ref, clear = res.labels, res.gap >= GAP_TOL
    assert np.array_equal(lab[clear], keep[ref][clear])


def test_assign_identity_anchor_is_cosine(pb):
    """ka = d and C_anchor = I: the half-step is cosine nearest-centroid (a textbook rule)."""
    d, N, ks = 64, 3000, 40
    w = random_qkv(1, 1, N, d, seed=9)
    ca = torch.eye(d)[None, None]
    cs = torch.randn(1, 1, ks, d, generator=torch.Generator().manual_seed(2))
    lab = pb.coclust_assign_step(w.q.cuda(), ca.cuda(), cs.cuda())[0, 0].cpu().numpy()
    X = f64(w.q[0, 0])
    C = cs[0, 0].double().numpy()
    cos = (X / np.linalg.norm(X, axis=1, keepdims=True)) @ (C / np.linalg.norm(C, axis=1, keepdims=True)).T
    srt = np.sort(cos, axis=1)
    clear = (srt[:, -1] - srt[:, -2]) > 1e-4
    assert np.array_equal(lab[clear], cos.argmax(1)[clear])


def test_assign_strided_bnhd_layout(pb):
    w = video_qkv(4, 8, 16, 3, 128, seed=4, layout="bnhd")
    assert w.k.stride(2) == 3 * 128
    ca = torch.randn(1, 3, 20, 128, generator=torch.Generator().manual_seed(0))
    cs = torch.randn(1, 3, 30, 128, generator=torch.Generator().manual_seed(1))
    lab = pb.coclust_assign_step(w.k.cuda(), ca.cuda(), cs.cuda()).cpu()
    lab2 = pb.coclust_assign_step(w.k.contiguous().cuda(), ca.cuda(), cs.cuda()).cpu()
    assert torch.equal(lab, lab2)
    for h in range(3):
        res = svoo.assign_step(f64(w.k[0, h]), ca[0, h].double().numpy(), cs[0, h].double().numpy())
        _check_labels(lab[0, h].numpy(), res)


# ------------------------------------------------------------------------- P4 selection
def _margins_ok(Cq, Ck, sq, sk, tau, d):
    A = Cq @ Ck.T
    for a in range(A.shape[0]):
        v = np.sort(A[a, sk > 0])[::-1]
        if len(v) > 1 and np.min(np.abs(np.diff(v)) / np.maximum(np.abs(v[:-1]), 1e-300)) < 1e-9:
            return False
        if sq[a] > 0:
            p = svoo.softmax_row(v / math.sqrt(d))
            if np.min(np.abs(np.cumsum(p) - (tau - 1e-12))) < 1e-12:
                return False
    return True


@pytest.mark.parametrize("rule", [svoo.RULE_DENSITY, svoo.RULE_AS_WRITTEN, svoo.RULE_FIXED])
@pytest.mark.parametrize("kq,kk,d,tau", [(16, 16, 64, 0.95), (100, 500, 128, 0.95), (7, 1024, 128, 0.9),
                                        (256, 1024, 128, 0.5), (1, 3, 64, 1.0)])
def test_block_select_bitexact(pb, rule, kq, kk, d, tau):
    H = 3
    budget = torch.tensor([0.05, 0.3, 0.97], dtype=torch.float32)
    theta = 0.1
    seed = kq * 7 + kk
    while True:
        g = torch.Generator().manual_seed(seed)
        Cq = torch.randn(1, H, kq, d, generator=g) * 0.3
        Ck = torch.randn(1, H, kk, d, generator=g) * 0.3
        sq = torch.randint(0, 3, (H, kq), generator=g)
        sk = torch.randint(0, 3, (H, kk), generator=g)
        sq[:, 0] = 1
        sk[:, 0] = 1
        if all(_margins_ok(Cq[0, h].double().numpy(), Ck[0, h].double().numpy(), sq[h].numpy(),
                           sk[h].numpy(), tau, d) for h in range(H)):
            break
        seed += 1000
    offs_q = torch.cat([torch.zeros(H, 1, dtype=torch.long), sq.cumsum(1)], 1).int()[None]
    offs_k = torch.cat([torch.zeros(H, 1, dtype=torch.long), sk.cumsum(1)], 1).int()[None]
    n_keep, kept = pb.block_select(Cq.cuda(), Ck.cuda(), offs_q.cuda(), offs_k.cuda(), budget.cuda(),
                                   tau, theta, rule)
    torch.cuda.synchronize()
    for h in range(H):
        ref = svoo.select_blocks(Cq[0, h].double().numpy(), Ck[0, h].double().numpy(), sq[h].numpy(),
                                 sk[h].numpy(), float(budget[h]), tau, theta, rule, d_head=d)
        assert n_keep[0, h].item() == ref.n_keep
        assert np.array_equal(kept[0, h, :, :ref.n_keep].cpu().numpy(), ref.kept)


def _margins_ok_z(Cq, Ck, sq, sk, tau, d, weighted):
    """_margins_ok on the ranking values of the NEXT-4 variants (z = Abar/sqrt(d) + log|K_c|)."""
    A = Cq @ Ck.T / math.sqrt(d) + (np.log(np.maximum(sk, 1)) if weighted else 0.0)
    for a in range(A.shape[0]):
        v = np.sort(A[a, sk > 0])[::-1]
        if len(v) > 1 and np.min(np.abs(np.diff(v)) / np.maximum(np.abs(v[:-1]), 1e-300)) < 1e-9:
            return False
        if sq[a] > 0:
            p = svoo.softmax_row(v)
            if np.min(np.abs(np.cumsum(p) - (tau - 1e-12))) < 1e-12:
                return False
    return True


@pytest.mark.parametrize("flags", [1, 2, 3])
@pytest.mark.parametrize("rule", [svoo.RULE_DENSITY, svoo.RULE_FIXED])
@pytest.mark.parametrize("kq,kk,d,tau", [(16, 16, 64, 0.95), (100, 500, 128, 0.95), (256, 1024, 128, 0.6)])
def test_block_select_variants_bitexact(pb, flags, rule, kq, kk, d, tau):
    """NEXT-4: per-row counts (R11b) and size-weighted importance (R9c): n_keep, the per-row
    counts and every kept row bit-exact against the oracle."""
    H = 3
    budget = torch.tensor([0.05, 0.3, 0.97], dtype=torch.float32)
    theta = 0.1
    seed = kq * 11 + kk + flags
    while True:
        g = torch.Generator().manual_seed(seed)
        Cq = torch.randn(1, H, kq, d, generator=g) * 0.3
        Ck = torch.randn(1, H, kk, d, generator=g) * 0.3
        sq = torch.randint(0, 4, (H, kq), generator=g)
        sk = torch.randint(0, 6, (H, kk), generator=g)
        sq[:, 0] = 1
        sk[:, 0] = 1
        if all(_margins_ok_z(Cq[0, h].double().numpy(), Ck[0, h].double().numpy(), sq[h].numpy(),
                             sk[h].numpy(), tau, d, flags & 2) for h in range(H)):
            break
        seed += 1000
    offs_q = torch.cat([torch.zeros(H, 1, dtype=torch.long), sq.cumsum(1)], 1).int()[None]
    offs_k = torch.cat([torch.zeros(H, 1, dtype=torch.long), sk.cumsum(1)], 1).int()[None]
    n_keep, kept, n_rows = pb.block_select(Cq.cuda(), Ck.cuda(), offs_q.cuda(), offs_k.cuda(), budget.cuda(),
                                           tau, theta, rule, flags=flags)
    torch.cuda.synchronize()
    for h in range(H):
        ref = svoo.select_blocks(Cq[0, h].double().numpy(), Ck[0, h].double().numpy(), sq[h].numpy(),
                                 sk[h].numpy(), float(budget[h]), tau, theta, rule, d_head=d,
                                 per_row=bool(flags & 1), size_weighted=bool(flags & 2))
        assert n_keep[0, h].item() == ref.n_keep
        rows = ref.n_rows if flags & 1 else np.full(kq, ref.n_keep)
        assert np.array_equal(n_rows[0, h].cpu().numpy(), rows)
        for a in range(kq):
            assert np.array_equal(kept[0, h, a, :rows[a]].cpu().numpy(), np.asarray(ref.kept[a]))


@pytest.mark.parametrize("kk", [300, 1000, 1024])
def test_block_select_exact_ties_and_float_collisions(pb, kk):
    """The selection order is (Abar desc, index asc) over exact float64 values (R11, R2).
    The kernel sorts 32-bit keys (value rounded to float, 22 bits) and puts colliding distinct
    values back into exact order; this case is built so that collisions and exact ties are the
    common case: Abar[a, j] = c_j + delta_j exactly (query rows e_0 + e_1, key rows (c_j, delta_j,
    0, ...)), c_j from a few float values and delta_j in {0, 1, 2, 3} * 2^-40, below half a float
    ulp of c_j — so every c_j group is one float key with up to four distinct doubles, each repeated
    (exact ties -> lower index).  Eight heads with the same rows and keep ratios spread over (0, 1)
    cut the order at many places; the FIXED kept sets pin the order, the DENSITY counts the
    recall prefix."""
    H, kq, d = 8, 3, 64
    g = torch.Generator().manual_seed(kk)
    cvals = torch.tensor([1.0, 1.5, 0.75, -0.5, 0.0, 1.25])
    c = cvals[torch.randint(0, len(cvals), (kk,), generator=g)]
    delta = torch.randint(0, 4, (kk,), generator=g).double() * 2.0 ** -40
    Ck = torch.zeros(kk, d, dtype=torch.float64)
    Ck[:, 0] = c.double()
    Ck[:, 1] = delta
    Cq = torch.zeros(kq, d, dtype=torch.float64)
    Cq[:, 0] = 1.0
    Cq[:, 1] = 1.0
    Cq[1, 0] = 2.0  # another exact row: 2 c_j + delta_j
    assert torch.equal(Ck.float().double(), Ck) and torch.equal(Cq.float().double(), Cq)
    sq = torch.ones(H, kq, dtype=torch.long)
    sk = torch.randint(1, 4, (H, kk), generator=g)
    sk[:, 5] = 0  # an empty key block is never eligible
    sk[:] = sk[0]
    offs_q = torch.cat([torch.zeros(H, 1, dtype=torch.long), sq.cumsum(1)], 1).int()[None]
    offs_k = torch.cat([torch.zeros(H, 1, dtype=torch.long), sk.cumsum(1)], 1).int()[None]
    budget = torch.tensor([0.01, 0.07, 0.13, 0.2, 0.33, 0.5, 0.77, 0.99], dtype=torch.float32)
    Cqh = Cq.float()[None, None].expand(1, H, kq, d).contiguous()
    Ckh = Ck.float()[None, None].expand(1, H, kk, d).contiguous()
    for rule in (svoo.RULE_FIXED, svoo.RULE_DENSITY):
        n_keep, kept = pb.block_select(Cqh.cuda(), Ckh.cuda(), offs_q.cuda(), offs_k.cuda(), budget.cuda(),
                                       0.9, 0.1, rule)
        torch.cuda.synchronize()
        for h in range(H):
            ref = svoo.select_blocks(Cq.numpy(), Ck.numpy(), sq[h].numpy(), sk[h].numpy(), float(budget[h]),
                                     0.9, 0.1, rule, d_head=d)
            assert n_keep[0, h].item() == ref.n_keep, (rule, h)
            assert np.array_equal(kept[0, h, :, :ref.n_keep].cpu().numpy(), ref.kept), (rule, h)


def test_attn_per_row_counts_and_fused_variants(pb):
    """Attention over per-row kept counts (R11b) against the oracle, and the fused entry with
    selection flags bit-equal to the staged entries."""
    w = video_qkv(6, 24, 40, 2, 128, seed=13)        # N = 5760
    kq, kk, iters, tau, theta = 40, 120, 2, 0.9, 0.1
    budget = torch.tensor([0.15, 0.35], dtype=torch.float32).cuda()
    q, k, v = w.q.cuda(), w.k.cuda(), w.v.cuda()
    for flags in (1, 3):
        st = pb.coclust_assign(q, k, kq, kk, iters, seed=3)
        n_keep, kept, n_rows = pb.block_select(st["cq"], st["ck"], st["offs_q"], st["offs_k"], budget, tau, theta,
                                               pb.RULE_DENSITY, flags=flags)
        o = pb.block_sparse_attn(q, k, v, st["perm_q"], st["offs_q"], st["perm_k"], st["offs_k"], n_keep, kept,
                                 n_keep_rows=n_rows)
        of = pb.coclust_sparse_attention(q, k, v, kq, kk, iters, budget, seed=3, tau=tau, theta=theta,
                                         rule=pb.RULE_DENSITY, sel_flags=flags)
        torch.cuda.synchronize()
        assert torch.equal(o, of)
        nr = n_rows.cpu().numpy()
        assert len(np.unique(nr)) > 1        # the rows really differ
        for h in range(2):
            rows = [kept[0, h, a, :nr[0, h, a]].cpu().numpy() for a in range(kq)]
            ref = svoo.sparse_attention(f64(w.q[0, h]), f64(w.k[0, h]), f64(w.v[0, h]),
                                        st["lq"][0, h].cpu().numpy(), st["lk"][0, h].cpu().numpy(), rows)
            err = np.abs(f64(o[0, h]) - ref)
            assert err.max() <= ATOL_MAX and err.mean() <= ATOL_MEAN


# ------------------------------------------------------------------------- P5 attention
def _oracle_state(w, kq, kk, seed, budget, rule, tau=0.95, theta=0.1, heads=None):
    """Run the oracle's co-clustering + selection per head; returns GPU-ready int32 tensors."""
    B, H, N, d = w.q.shape
    heads = range(H) if heads is None else heads
    st = dict(perm_q=[], offs_q=[], perm_k=[], offs_k=[], n_keep=[], kept=[], Lq=[], Lk=[], sel=[])
    for h in heads:
        Q, K = f64(w.q[0, h]), f64(w.k[0, h])
        cc = svoo.cocluster(Q, K, kq, kk, 2, seed=seed, h=h, H=H)
        pq, oq = svoo.counting_sort(cc.Lq, kq)
        pk, ok = svoo.counting_sort(cc.Lk, kk)
        sel = svoo.select_blocks(cc.Cq, cc.Ck, np.diff(oq), np.diff(ok), budget, tau, theta, rule, d_head=d)
        kept = np.full((kq, kk), -1, np.int64)
        kept[:, :sel.n_keep] = sel.kept
        for key, val in (("perm_q", pq), ("offs_q", oq), ("perm_k", pk), ("offs_k", ok), ("kept", kept)):
            st[key].append(torch.from_numpy(val.astype(np.int32)))
        st["n_keep"].append(sel.n_keep)
        st["Lq"].append(cc.Lq); st["Lk"].append(cc.Lk); st["sel"].append(sel)
    g = {k: torch.stack(st[k])[None].cuda() for k in ("perm_q", "offs_q", "perm_k", "offs_k", "kept")}
    g["n_keep"] = torch.tensor(st["n_keep"], dtype=torch.int32)[None].cuda()
    return g, st


def _attn_check(O_gpu, w, st, h):
    Q, K, V = f64(w.q[0, h]), f64(w.k[0, h]), f64(w.v[0, h])
    ref = svoo.sparse_attention(Q, K, V, st["Lq"][h], st["Lk"][h], st["sel"][h].kept)
    err = np.abs(f64(O_gpu[0, h]) - ref)
    assert err.max() <= ATOL_MAX, err.max()
    assert err.mean() <= ATOL_MEAN, err.mean()
    return err.max(), err.mean()


def _one_row(Q, K, V, Lq, Lk, kept, i):
    allowed = np.nonzero(np.isin(Lk, kept[Lq[i]]))[0]
    s = (K[allowed] @ Q[i]) / math.sqrt(Q.shape[1])
    e = np.exp(s - s.max())
    return (e @ V[allowed]) / e.sum()


@pytest.mark.parametrize("cfg", ["toy", "mid", "mid_dense"])
def test_block_sparse_attn(pb, cfg):
    if cfg == "toy":
        w = config_workload("toy")
        kq, kk, budget, rule = 16, 16, 0.3, svoo.RULE_DENSITY
    else:
        w = video_qkv(6, 24, 40, 2, 128, seed=11)        # N = 5760 (45 tiles, ragged clusters)
        kq, kk = 40, 120
        budget, rule = (1.0, svoo.RULE_FIXED) if cfg == "mid_dense" else (0.2, svoo.RULE_FIXED)
    g, st = _oracle_state(w, kq, kk, 0, budget, rule)
    O = pb.block_sparse_attn(w.q.cuda(), w.k.cuda(), w.v.cuda(), g["perm_q"], g["offs_q"], g["perm_k"],
                             g["offs_k"], g["n_keep"], g["kept"])
    torch.cuda.synchronize()
    for h in range(w.q.shape[1]):
        _attn_check(O, w, st, h)
    if cfg == "mid_dense":   # keep ratio 1.0 == dense softmax attention
        for h in range(w.q.shape[1]):
            ref = svoo.dense_attention(f64(w.q[0, h]), f64(w.k[0, h]), f64(w.v[0, h]))
            assert np.abs(f64(O[0, h]) - ref).max() <= ATOL_MAX


def test_attn_tiny_clusters_and_single_query_cluster(pb):
    """Clusters smaller than one 8-row unit, a single query cluster, N not a multiple of 128."""
    d, N = 64, 300
    w = random_qkv(1, 1, N, d, seed=21)
    Lq = np.zeros(N, np.int64)                         # one query cluster of 300 rows (3 tiles)
    Lk = np.random.default_rng(0).integers(0, 90, N)   # ~3.3 keys per key cluster
    pq, oq = svoo.counting_sort(Lq, 1)
    pk, ok = svoo.counting_sort(Lk, 90)
    ne = np.nonzero(np.diff(ok) > 0)[0]
    kept = np.full((1, 90), -1, np.int64)
    sel = ne[::3]
    kept[0, :len(sel)] = sel
    t = lambda a: torch.from_numpy(a.astype(np.int32))[None, None].cuda()
    O = pb.block_sparse_attn(w.q.cuda(), w.k.cuda(), w.v.cuda(), t(pq), t(oq), t(pk), t(ok),
                             torch.tensor([[len(sel)]], dtype=torch.int32).cuda(),
                             torch.from_numpy(kept.astype(np.int32))[None, None].cuda())
    ref = svoo.sparse_attention(f64(w.q[0, 0]), f64(w.k[0, 0]), f64(w.v[0, 0]), Lq, Lk, [sel])
    err = np.abs(f64(O[0, 0]) - ref)
    assert err.max() <= ATOL_MAX and err.mean() <= ATOL_MEAN


@pytest.mark.parametrize("d", [64, 128])
def test_attn_split_kv_single_tile_items(pb, d):
    """Work items with one query tile run split-KV (even / odd KV tiles on the two accumulator
    sets, merged in the epilogue).  Query clusters of 1..4 tiles (single, pair, pair + single)
    against kept key sets of 1..9 KV tiles (odd and even counts, one tile only)."""
    rng = np.random.default_rng(5)
    q_sizes = [60, 128, 129, 300, 1, 500, 77, 255]
    k_sizes = [3, 5, 130, 64, 200, 1, 90, 257, 40, 128, 33, 400, 8, 16, 300, 7]
    N = max(sum(q_sizes), sum(k_sizes))
    q_sizes[-1] += N - sum(q_sizes)
    k_sizes[-1] += N - sum(k_sizes)
    kq, kk = len(q_sizes), len(k_sizes)
    Lq = rng.permutation(np.repeat(np.arange(kq), q_sizes))
    Lk = rng.permutation(np.repeat(np.arange(kk), k_sizes))
    w = random_qkv(1, 1, N, d, seed=31)
    pq, oq = svoo.counting_sort(Lq, kq)
    pk, ok = svoo.counting_sort(Lk, kk)
    n_keep = 4
    kept = np.full((kq, kk), -1, np.int64)
    sel = []
    for a in range(kq):
        if a == 0:
            ka = np.array([0, 1, 5, 12])                 # 17 keys -> a single KV tile
        elif a == 1:
            ka = np.array([0, 2, 5, 12])                 # 144 keys -> two KV tiles
        else:
            ka = np.sort(rng.choice(kk, n_keep, replace=False))
        kept[a, :n_keep] = ka
        sel.append(ka)
    t = lambda x: torch.from_numpy(x.astype(np.int32))[None, None].cuda()
    O = pb.block_sparse_attn(w.q.cuda(), w.k.cuda(), w.v.cuda(), t(pq), t(oq), t(pk), t(ok),
                             torch.tensor([[n_keep]], dtype=torch.int32).cuda(),
                             torch.from_numpy(kept.astype(np.int32))[None, None].cuda())
    ref = svoo.sparse_attention(f64(w.q[0, 0]), f64(w.k[0, 0]), f64(w.v[0, 0]), Lq, Lk, sel)
    err = np.abs(f64(O[0, 0]) - ref)
    assert err.max() <= ATOL_MAX and err.mean() <= ATOL_MEAN, (err.max(), err.mean())


def test_attn_singleton_keys_pick_value(pb):
    """singleton key blocks, one kept block per query block -> o_i = v_{j*}."""
    d, N = 128, 256
    w = random_qkv(1, 1, N, d, seed=5)
    Lq = np.arange(N) % 4
    Lk = np.arange(N)
    pq, oq = svoo.counting_sort(Lq, 4)
    pk, ok = svoo.counting_sort(Lk, N) if N <= 1024 else None
    kept = np.full((4, N), -1, np.int64)
    kept[:, 0] = [3, 77, 150, 255]
    t = lambda a: torch.from_numpy(np.asarray(a).astype(np.int32))
    O = pb.block_sparse_attn(w.q.cuda(), w.k.cuda(), w.v.cuda(), t(pq)[None, None].cuda(),
                             t(oq)[None, None].cuda(), t(pk)[None, None].cuda(), t(ok)[None, None].cuda(),
                             torch.ones(1, 1, dtype=torch.int32).cuda(), t(kept)[None, None].cuda())
    exp = w.v[0, 0][torch.tensor([3, 77, 150, 255])[Lq]]
    assert torch.equal(O[0, 0].cpu(), exp)


@pytest.mark.parametrize("order", ["rising", "falling"])
def test_attn_max_jumps_within_tiles(pb, order):
    """The online softmax's rescaling paths (attn.cu: P(j) is computed against the running max of
    the earlier tiles; a tile whose max grows by > 8 in the log2 domain moves the reference for the
    next tile; a jump so large that a P half's row sum would exceed 2^40 is recomputed mid-tile,
    in the first or the second 64-key half).  One key cluster of 1024 keys in token order (8 key
    tiles); the score level q.k ~ 128 g steps up inside tile 1's second half (g = 3, a jump of ~49
    in the log2 domain), at tile 2's first half (g = 6), by a moderate 0.7 at tile 4 (~11), and is
    random below the maximum afterwards.  Query clusters of 100 rows (one split-KV item) and 924
    rows (pair items plus one split-KV item); every query keeps the only key cluster."""
    d, N = 128, 1024
    gen = torch.Generator().manual_seed(11)
    g = np.zeros(N)
    g[192:256] = 3.0
    g[256:512] = 6.0
    g[512:640] = 6.7
    g[640:] = np.random.default_rng(3).uniform(0.0, 6.7, N - 640)
    if order == "falling":
        g = g[::-1].copy()
    u = torch.ones(d)
    q = (u + 0.5 * torch.randn(N, d, generator=gen)).to(torch.bfloat16)
    k = (torch.from_numpy(g).float()[:, None] * u + 0.3 * torch.randn(N, d, generator=gen)).to(torch.bfloat16)
    v = torch.randn(N, d, generator=gen).to(torch.bfloat16)
    Lq = np.where(np.arange(N) % 10 == 0, 0, 1)  # 103 / 921 rows
    Lk = np.zeros(N, np.int64)
    pq, oq = svoo.counting_sort(Lq, 2)
    pk, ok = svoo.counting_sort(Lk, 1)
    kept = np.zeros((2, 1), np.int64)
    t = lambda a: torch.from_numpy(np.asarray(a).astype(np.int32))
    O = pb.block_sparse_attn(q[None, None].cuda(), k[None, None].cuda(), v[None, None].cuda(),
                             t(pq)[None, None].cuda(), t(oq)[None, None].cuda(), t(pk)[None, None].cuda(),
                             t(ok)[None, None].cuda(), torch.ones(1, 1, dtype=torch.int32).cuda(),
                             t(kept)[None, None].cuda())
    ref = svoo.sparse_attention(f64(q), f64(k), f64(v), Lq, Lk, kept)
    err = np.abs(f64(O[0, 0]) - ref)
    assert np.isfinite(f64(O[0, 0])).all()
    assert err.max() <= ATOL_MAX and err.mean() <= ATOL_MEAN, (err.max(), err.mean())


# ------------------------------------------------------------------------- P6 end to end
def test_fused_toy_end_to_end(pb):
    """P6 on the toy config: the first sampler seed whose oracle run has no near-tie in any
    half-step (every gap >= 1e-4; seeds 3 and 14 of the first 60 qualify) must give identical
    labels end to end and an output within P5.  Seeds with near-ties are covered by the chained
    teacher-forced tests."""
    w = config_workload("toy")
    Q, K, V = f64(w.q[0, 0]), f64(w.k[0, 0]), f64(w.v[0, 0])
    seed = ref = None
    for s_ in range(60):
        r_ = svoo.coclust_sparse_attention_head(Q, K, V, 16, 16, 3, s_, 0.3, 0.95, 0.1, svoo.RULE_DENSITY)
        if min(float(np.min(t["gap"])) for t in r_.cc.trace) >= GAP_TOL:
            seed, ref = s_, r_
            break
    assert seed is not None, "no near-tie-free toy seed in 0..59"
    budget = torch.tensor([0.3], dtype=torch.float32)
    r = pb.coclust_assign(w.q.cuda(), w.k.cuda(), 16, 16, 3, seed=seed)
    O = pb.coclust_sparse_attention(w.q.cuda(), w.k.cuda(), w.v.cuda(), 16, 16, 3, budget.cuda(), seed=seed)
    torch.cuda.synchronize()
    assert np.array_equal(r["lq"][0, 0].cpu().numpy(), ref.cc.Lq)
    assert np.array_equal(r["lk"][0, 0].cpu().numpy(), ref.cc.Lk)
    assert np.array_equal(r["perm_q"][0, 0].cpu().numpy(), ref.perm_q)
    assert np.array_equal(r["offs_k"][0, 0].cpu().numpy(), ref.offs_k)
    err = np.abs(f64(O[0, 0]) - ref.O)
    assert err.max() <= ATOL_MAX and err.mean() <= ATOL_MEAN


@pytest.mark.parametrize("T,Hs,Ws,kq,kk", [(4, 8, 16, 12, 20), (1, 8, 8, 48, 60), (1, 10, 10, 100, 100),
                                        (1, 30, 50, 700, 1024), (2, 16, 32, 1000, 1024)])
def test_sampler_matches_oracle_via_explicit_init(pb, T, Hs, Ws, kq, kk):
    """coclust_assign(seed) == coclust_assign(init = oracle's R4 sample): pins the GPU sampler,
    including collision-heavy draws (K close to N: Floyd's j_i picks and draws t_i >= N - K)."""
    w = video_qkv(T, Hs, Ws, 2, 64, seed=3)
    N = w.q.shape[2]
    iq = np.stack([svoo.sample_anchor_indices(N, kq, 99, 0, h, 2, 0) for h in range(2)])[None]
    ik = np.stack([svoo.sample_anchor_indices(N, kk, 99, 0, h, 2, 1) for h in range(2)])[None]
    a = pb.coclust_assign(w.q.cuda(), w.k.cuda(), kq, kk, 1, seed=99)
    b = pb.coclust_assign(w.q.cuda(), w.k.cuda(), kq, kk, 1, seed=12345,
                          init_q=torch.from_numpy(iq.astype(np.int32)).cuda(),
                          init_k=torch.from_numpy(ik.astype(np.int32)).cuda())
    for key in a:
        assert torch.equal(a[key], b[key]), key


def test_coclust_assign_chain_teacher_forced(pb):
    """Each GPU half-step matches the oracle's half-step given the oracle's centroids (P1, chained)."""
    w = video_qkv(8, 16, 24, 1, 128, seed=8)
    Q, K = f64(w.q[0, 0]), f64(w.k[0, 0])
    cc = svoo.cocluster(Q, K, 40, 120, 2, seed=0)
    for t in cc.trace:
        X = w.k if t["side"] == "k" else w.q
        ca = torch.from_numpy(t["C_anchor"]).float()[None, None].cuda()
        cs = torch.from_numpy(t["C_self"]).float()[None, None].cuda()
        lab = pb.coclust_assign_step(X.cuda(), ca, cs)[0, 0].cpu().numpy()
        ok = t["gap"] >= GAP_TOL
        assert np.sum((lab != t["labels"]) & ok) == 0


def test_determinism_and_head_sharding(pb):
    """Bitwise-identical reruns, and a head-sharded call (head_offset/heads_total) reproduces the
    single call's heads bit for bit (kernels are per head; R4 streams are keyed by global head)."""
    w = video_qkv(4, 16, 32, 4, 128, seed=1)
    budget = torch.tensor([0.2, 0.4, 0.3, 0.1], dtype=torch.float32).cuda()
    q, k, v = w.q.cuda(), w.k.cuda(), w.v.cuda()
    o1 = pb.coclust_sparse_attention(q, k, v, 20, 60, 2, budget)
    o2 = pb.coclust_sparse_attention(q, k, v, 20, 60, 2, budget)
    assert torch.equal(o1, o2)
    for r in range(2):
        sl = slice(2 * r, 2 * r + 2)
        o3 = pb.coclust_sparse_attention(q[:, sl].contiguous(), k[:, sl].contiguous(), v[:, sl].contiguous(),
                                         20, 60, 2, budget[sl].contiguous(), head_offset=2 * r, heads_total=4)
        assert torch.equal(o3, o1[:, sl])


def test_clustering_reuse_cached_entry(pb):
    """NEXT-1: recompute=True == the fused layer and fills the state; recompute=False
    reuses the stored labels / kept blocks on new inputs (checked against the oracle)."""
    w = video_qkv(4, 16, 24, 2, 128, seed=6)
    q, k, v = w.q.cuda(), w.k.cuda(), w.v.cuda()
    budget = torch.tensor([0.25, 0.35], dtype=torch.float32).cuda()
    B, H, N, d = q.shape
    st = pb.LayerState(B, H, N, d, 24, 64, q.device)
    o_full = pb.coclust_sparse_attention(q, k, v, 24, 64, 2, budget)
    o_rec = pb.coclust_sparse_attention_cached(q, k, v, 24, 64, 2, budget, st, True)
    ref = pb.coclust_assign(q, k, 24, 64, 2)
    torch.cuda.synchronize()
    assert torch.equal(o_full, o_rec)
    for key in ("lq", "lk", "perm_q", "offs_q", "perm_k", "offs_k"):
        assert torch.equal(getattr(st, key), ref[key]), key
    o_same = pb.coclust_sparse_attention_cached(q, k, v, 24, 64, 2, budget, st, False)
    assert torch.equal(o_same, o_full)
    g = torch.Generator(device="cuda").manual_seed(1)
    q2 = (q.float() + 0.05 * torch.randn(q.shape, generator=g, device="cuda")).to(torch.bfloat16)
    v2 = (v.float() + 0.05 * torch.randn(v.shape, generator=g, device="cuda")).to(torch.bfloat16)
    o2 = pb.coclust_sparse_attention_cached(q2, k, v2, 24, 64, 2, budget, st, False)
    torch.cuda.synchronize()
    for h in range(H):
        n = int(st.n_keep[0, h])
        ref_o = svoo.sparse_attention(f64(q2[0, h]), f64(k[0, h]), f64(v2[0, h]), st.lq[0, h].cpu().numpy(),
                                      st.lk[0, h].cpu().numpy(), st.kept[0, h, :, :n].cpu().numpy())
        err = np.abs(f64(o2[0, h]) - ref_o)
        assert err.max() <= ATOL_MAX and err.mean() <= ATOL_MEAN


# ------------------------------------------------------------------------- NEXT-2 k-means baseline
@pytest.mark.parametrize("d,N,ks", [(64, 2048, 16), (128, 8192, 500), (128, 3000, 100), (128, 4096, 1024),
                                    (64, 3000, 300),
                                    (64, 1000, 1)])
def test_kmeans_assign_step(pb, d, N, ks):
    """k-means half-step through the assignment GEMM with the -||c||^2/2 bias epilogue: labels
    identical to the oracle's argmin_j ||x_i - c_j|| outside the near-tie band (P1 rule)."""
    w = video_qkv(4, 16, max(1, N // 64), 2, d, seed=ks + 3)
    g = torch.Generator().manual_seed(ks)
    C = torch.randn(1, 2, ks, d, generator=g) * 0.8
    for X in (w.q, w.k):
        lab = pb.kmeans_assign_step(X.cuda(), C.cuda()).cpu()
        for h in range(2):
            res = svoo.kmeans_step(f64(X[0, h]), C[0, h].double().numpy())
            _check_labels(lab[0, h].numpy(), res, "kmeans")


def test_kmeans_assign_chain_teacher_forced_and_layer(pb):
    """Every GPU k-means half-step matches the oracle given the oracle's centroids; the whole
    "w/o On" layer (CLUSTER_KMEANS) equals the staged entries bit for bit and the oracle within P5."""
    w = video_qkv(8, 16, 24, 1, 128, seed=9)
    Q, K = f64(w.q[0, 0]), f64(w.k[0, 0])
    cc = svoo.cocluster_kmeans(Q, K, 40, 120, 2, seed=0)
    for t in cc.trace:
        X = w.k if t["side"] == "k" else w.q
        cs = torch.from_numpy(t["C_self"]).float()[None, None].cuda()
        lab = pb.kmeans_assign_step(X.cuda(), cs)[0, 0].cpu().numpy()
        ok = t["gap"] >= GAP_TOL
        assert np.sum((lab != t["labels"]) & ok) == 0
    q, k, v = w.q.cuda(), w.k.cuda(), w.v.cuda()
    budget = torch.tensor([0.3], dtype=torch.float32).cuda()
    st = pb.coclust_assign(q, k, 40, 120, 2, seed=0, kmeans=True)
    n_keep, kept = pb.block_select(st["cq"], st["ck"], st["offs_q"], st["offs_k"], budget, 0.95, 0.1,
                                   pb.RULE_DENSITY)
    o = pb.block_sparse_attn(q, k, v, st["perm_q"], st["offs_q"], st["perm_k"], st["offs_k"], n_keep, kept)
    of = pb.coclust_sparse_attention(q, k, v, 40, 120, 2, budget, seed=0, sel_flags=pb.CLUSTER_KMEANS)
    torch.cuda.synchronize()
    assert torch.equal(o, of)
    n = int(n_keep[0, 0])
    ref = svoo.sparse_attention(Q, K, f64(w.v[0, 0]), st["lq"][0, 0].cpu().numpy(), st["lk"][0, 0].cpu().numpy(),
                                kept[0, 0, :, :n].cpu().numpy())
    err = np.abs(f64(o[0, 0]) - ref)
    assert err.max() <= ATOL_MAX and err.mean() <= ATOL_MEAN
    # every nonempty centroid is the mean of its members (P2 on the k-means side)
    for side, X, L, C in (("k", K, st["lk"], st["ck"]), ("q", Q, st["lq"], st["cq"])):
        Lh, Ch = L[0, 0].cpu().numpy(), C[0, 0].cpu().double().numpy()
        for j in np.unique(Lh):
            m = X[Lh == j].mean(0)
            assert np.allclose(Ch[j], m, rtol=1e-5, atol=1e-5), side


def test_streamed_layer_matches_direct_calls(pb):
    """runtime.StreamedLayer (upload / layer / download on three streams, two buffer sets) returns
    exactly the outputs of direct calls, for more calls than buffer sets."""
    from paper_2603_18636_b200.runtime import StreamedLayer
    budget = torch.tensor([0.3, 0.5], dtype=torch.float32).cuda()
    ins = [video_qkv(4, 16, 16, 2, 128, seed=40 + i) for i in range(5)]
    ref = [pb.coclust_sparse_attention(w.q.cuda(), w.k.cuda(), w.v.cuda(), 12, 40, 2, budget).cpu() for w in ins]
    pinned = [tuple(t.pin_memory() for t in (w.q, w.k, w.v)) for w in ins]
    outs = [torch.empty_like(ins[0].q).pin_memory() for _ in ins]
    ws = pb.Workspace()
    sl = StreamedLayer(lambda dq, dk, dv, do: pb.coclust_sparse_attention(dq, dk, dv, 12, 40, 2, budget, out=do,
                                                                         ws=ws),
                       ins[0].q.shape, "cuda", depth=2)
    for i, (hq, hk, hv) in enumerate(pinned):
        sl.submit(i, hq, hk, hv, outs[i])
    torch.cuda.synchronize()
    for o, r in zip(outs, ref):
        assert torch.equal(o, r)


def test_layer_cuda_graph_capture_and_replay(pb):
    """The whole layer enqueues only device work on the caller's stream (no host round trip), so
    it captures into a CUDA graph; replays with new inputs copied into the captured buffers equal
    eager calls bit for bit (stage-event records inside the graph included; CUDA does not time
    events recorded by graph replays, so graph runs are timed around the replay)."""
    budget = torch.tensor([0.3, 0.5], dtype=torch.float32).cuda()
    w0, w1 = video_qkv(4, 16, 16, 2, 128, seed=50), video_qkv(4, 16, 16, 2, 128, seed=51)
    q, k, v = (t.cuda() for t in (w0.q, w0.k, w0.v))
    out = torch.empty_like(q)
    ws = pb.Workspace()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    for e in evs:
        e.record()  # torch creates the CUDA event lazily, on first record
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(2):  # warm-up: workspace allocation and kernel attributes outside capture
            pb.coclust_sparse_attention(q, k, v, 12, 40, 2, budget, out=out, ws=ws, stage_events=evs)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        pb.coclust_sparse_attention(q, k, v, 12, 40, 2, budget, out=out, ws=ws, stage_events=evs)
    for w in (w1, w0):
        q.copy_(w.q), k.copy_(w.k), v.copy_(w.v)
        g.replay()
        torch.cuda.synchronize()
        ref = pb.coclust_sparse_attention(w.q.cuda(), w.k.cuda(), w.v.cuda(), 12, 40, 2, budget)
        torch.cuda.synchronize()
        assert torch.equal(out, ref)


@pytest.mark.parametrize("kk", [48, 200])  # 200: the CTA-pair assignment kernel over (b, h) units
def test_batch_of_two_layers(pb, kk):
    """B = 2: the sampler streams are keyed by b (R4: (b H + h) 2 + side), every kernel indexes
    (b, h) through the strides.  First-iteration labels of batch 1 match the oracle run with b = 1
    (outside near-ties), and each (b, h) output matches the oracle's masked attention on the GPU's
    own partition."""
    d = 128
    w = random_qkv(2, 2, 1500, d, seed=61)
    q, k, v = w.q.cuda(), w.k.cuda(), w.v.cuda()
    st = pb.coclust_assign(q, k, 16, kk, 1, seed=4)
    torch.cuda.synchronize()
    for b in range(2):
        for h in range(2):
            cc = svoo.cocluster(f64(w.q[b, h]), f64(w.k[b, h]), 16, kk, 1, seed=4, b=b, h=h, H=2)
            tk = cc.trace[0]
            ok = tk["gap"] >= GAP_TOL
            assert np.sum((st["lk"][b, h].cpu().numpy() != tk["labels"]) & ok) == 0, (b, h)
    budget = torch.tensor([0.3, 0.5], dtype=torch.float32).cuda()
    st = pb.coclust_assign(q, k, 16, kk, 2, seed=4)
    n_keep, kept = pb.block_select(st["cq"], st["ck"], st["offs_q"], st["offs_k"], budget, 0.95, 0.1, pb.RULE_DENSITY)
    o = pb.block_sparse_attn(q, k, v, st["perm_q"], st["offs_q"], st["perm_k"], st["offs_k"], n_keep, kept)
    of = pb.coclust_sparse_attention(q, k, v, 16, kk, 2, budget, seed=4)
    torch.cuda.synchronize()
    assert torch.equal(o, of)
    for b in range(2):
        for h in range(2):
            n = int(n_keep[b, h])
            ref = svoo.sparse_attention(f64(w.q[b, h]), f64(w.k[b, h]), f64(w.v[b, h]), st["lq"][b, h].cpu().numpy(),
                                        st["lk"][b, h].cpu().numpy(), kept[b, h, :, :n].cpu().numpy())
            err = np.abs(f64(o[b, h]) - ref)
            assert err.max() <= ATOL_MAX and err.mean() <= ATOL_MEAN, (b, h, err.max())


def test_attn_many_small_clusters_1024(pb):
    """K_q = K_k = 1024 (the ABI maximum) on N = 8192: query clusters of ~8 rows (every item a
    single-tile split-KV item), key clusters of ~8 keys (one 8-row unit each, heavy masking).
    The whole layer against the oracle's masked attention on the GPU's partition."""
    w = video_qkv(4, 32, 64, 1, 128, seed=80)
    q, k, v = w.q.cuda(), w.k.cuda(), w.v.cuda()
    budget = torch.tensor([0.15], dtype=torch.float32).cuda()
    st = pb.coclust_assign(q, k, 1024, 1024, 2, seed=1)
    n_keep, kept = pb.block_select(st["cq"], st["ck"], st["offs_q"], st["offs_k"], budget, 0.95, 0.1, pb.RULE_FIXED)
    o = pb.coclust_sparse_attention(q, k, v, 1024, 1024, 2, budget, seed=1, rule=pb.RULE_FIXED)
    torch.cuda.synchronize()
    n = int(n_keep[0, 0])
    assert n == 154
    ref = svoo.sparse_attention(f64(w.q[0, 0]), f64(w.k[0, 0]), f64(w.v[0, 0]), st["lq"][0, 0].cpu().numpy(),
                                st["lk"][0, 0].cpu().numpy(), kept[0, 0, :, :n].cpu().numpy())
    err = np.abs(f64(o[0, 0]) - ref)
    assert err.max() <= ATOL_MAX and err.mean() <= ATOL_MEAN, (err.max(), err.mean())
