"""Pins for the float64 oracle (oracle/svoo.py) against things other than itself:
the paper/SPEC worked examples (tests/golden), published test vectors, closed forms, library
routines (scipy / torch SDPA / np.argsort) and brute force on tiny inputs.  CPU only."""
import itertools
import json
import math
import os

import numpy as np
import pytest
import torch

from oracle import svoo

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


# ---------------------------------------------------------------- sampler (R4)
def test_splitmix64_published_vector():
    for case in GOLD["splitmix64"]:
        s = case["seed"]
        outs = []
        for _ in range(len(case["out"])):
            s, o = svoo.splitmix64_next(s)
            outs.append(str(o))
        assert outs == case["out"], case["cite"]


@pytest.mark.parametrize("N,K", [(10, 10), (100, 1), (2048, 16), (5000, 1024)])
def test_sample_distinct_sorted_in_range(N, K):
    idx = svoo.sample_anchor_indices(N, K, seed=7, b=0, h=3, H=4, side=1)
    assert idx.shape == (K,)
    assert np.all(np.diff(idx) > 0)
    assert idx[0] >= 0 and idx[-1] < N
    if K == N:
        assert np.array_equal(idx, np.arange(N))


def test_sample_uniform_and_stream_separation():
    N, K, T = 20, 5, 4000
    cnt = np.zeros(N)
    for s in range(T):
        cnt[svoo.sample_anchor_indices(N, K, seed=s, b=0, h=0, H=1, side=0)] += 1
    expected = T * K / N
    chi2 = ((cnt - expected) ** 2 / expected).sum()
    assert chi2 < 50, chi2          # 19 dof: p(chi2 > 50) ~ 1e-4
    a = svoo.sample_anchor_indices(1000, 50, 1, 0, 0, 2, 0)
    b = svoo.sample_anchor_indices(1000, 50, 1, 0, 0, 2, 1)
    c = svoo.sample_anchor_indices(1000, 50, 1, 0, 1, 2, 0)
    assert not np.array_equal(a, b) and not np.array_equal(a, c)


# ---------------------------------------------------------------- numerics (golden)
def test_softmax_golden():
    for case in GOLD["softmax"]:
        np.testing.assert_allclose(svoo.softmax_row(case["in"]), case["out"], rtol=0, atol=1e-15)


def test_softmax_matches_scipy_and_shift_invariance():
    from scipy.special import softmax
    z = np.random.default_rng(0).normal(size=50) * 30
    np.testing.assert_allclose(svoo.softmax_row(z), softmax(z), rtol=1e-13, atol=0)
    np.testing.assert_allclose(svoo.softmax_row(z + 700), svoo.softmax_row(z), rtol=1e-12)


def test_l2_normalize_golden():
    for case in GOLD["l2_normalize"]:
        np.testing.assert_allclose(svoo.l2_normalize_rows(case["in"]), case["out"], atol=1e-15)


# ---------------------------------------------------------------- assignment (Alg. 1 Step A/B)
def _explicit_distance_labels(X, Ca, Cs):
    """Brute force: normalise with Python loops and compute ||a-b|| by explicit differences."""
    def norm_rows(M):
        out = []
        for r in M:
            n = math.sqrt(sum(float(v) * float(v) for v in r))
            out.append([float(v) / n for v in r] if n > 0 else [float(v) for v in r])
        return out
    P = norm_rows([[sum(float(x[t]) * float(c[t]) for t in range(len(x))) for c in Ca] for x in X])
    Pb = norm_rows([[sum(float(s[t]) * float(c[t]) for t in range(len(s))) for c in Ca] for s in Cs])
    labels, dists = [], []
    for p in P:
        D = [math.sqrt(sum((p[t] - q[t]) ** 2 for t in range(len(p)))) for q in Pb]
        best = min(range(len(D)), key=lambda j: (D[j], j))
        labels.append(best)
        dists.append(D)
    return np.array(labels), np.array(dists)


def test_assign_matches_explicit_differences():
    rng = np.random.default_rng(1)
    X, Ca, Cs = rng.normal(size=(40, 6)), rng.normal(size=(5, 6)), rng.normal(size=(7, 6))
    r = svoo.assign_step(X, Ca, Cs)
    lab, D = _explicit_distance_labels(X, Ca, Cs)
    assert np.array_equal(r.labels, lab)
    np.testing.assert_allclose(r.dist_best, D[np.arange(40), lab], atol=1e-12)


def test_assign_identity_anchor_is_cosine_nearest_centroid():
    """With C_anchor = I_d the step is the textbook cosine nearest-centroid rule (sklearn)."""
    from sklearn.metrics.pairwise import cosine_similarity
    rng = np.random.default_rng(2)
    d = 16
    X, Cs = rng.normal(size=(500, d)), rng.normal(size=(12, d))
    r = svoo.assign_step(X, np.eye(d), Cs)
    assert np.array_equal(r.labels, cosine_similarity(X, Cs).argmax(1))


def test_assign_single_cluster_and_ties():
    rng = np.random.default_rng(3)
    X = rng.normal(size=(30, 4))
    assert np.all(svoo.assign_step(X, rng.normal(size=(3, 4)), rng.normal(size=(1, 4))).labels == 0)
    Cs = np.stack([np.ones(4), np.ones(4), -np.ones(4)])  # clusters 0 and 1 identical -> ties to 0
    r = svoo.assign_step(X, np.eye(4), Cs)
    assert not np.any(r.labels == 1)


def test_reduced_form_agrees_with_literal():
    """SURVEY §8c reduced form: argmin_j ||P^_i - Pbar^_j|| == argmax_j x_i . W_j,
    W_j = Gamma c_j / ||Pbar_j||, Gamma = C_a^T C_a.  A different algebraic route (the one the
    CUDA kernel uses), so a dropped normalisation or transposed operand in the oracle fails."""
    rng = np.random.default_rng(4)
    X, Ca, Cs = rng.normal(size=(3000, 32)), rng.normal(size=(20, 32)), rng.normal(size=(50, 32))
    r = svoo.assign_step(X, Ca, Cs)
    G = Ca.T @ Ca
    W = (G @ Cs.T) / np.linalg.norm(Cs @ Ca.T, axis=1)[None, :]
    red = (X @ W).argmax(1)
    ok = r.gap > 1e-9
    assert np.array_equal(r.labels[ok], red[ok])


def test_planted_two_groups_bruteforce():
    """n=8 keys in two well-separated groups, K=2: Step A recovers the planted partition, and
    it is the best of all 2-partitions under the normalised-affinity scatter (brute force)."""
    rng = np.random.default_rng(5)
    d = 8
    g0, g1 = rng.normal(size=d) * 3, rng.normal(size=d) * 3
    truth = np.array([0, 0, 0, 0, 1, 1, 1, 1])
    K = np.stack([(g0 if t == 0 else g1) + 0.05 * rng.normal(size=d) for t in truth])
    Q = K + 0.05 * rng.normal(size=K.shape)
    res = svoo.cocluster(Q, K, 2, 2, 3, init_q=np.array([0, 4]), init_k=np.array([1, 5]))
    for lab in (res.Lk, res.Lq):
        assert np.array_equal(lab, truth) or np.array_equal(lab, 1 - truth)
    P = svoo.l2_normalize_rows(K @ res.Cq.T)

    def scatter(lab):
        s = 0.0
        for c in (0, 1):
            m = P[lab == c]
            if len(m):
                s += ((m - m.mean(0)) ** 2).sum()
        return s
    best = min((scatter(np.array(bits)), bits) for bits in itertools.product((0, 1), repeat=8)
               if 0 < sum(bits) < 8)
    assert np.array_equal(np.array(best[1]), truth) or np.array_equal(np.array(best[1]), 1 - truth)


# ---------------------------------------------------------------- centroid update
def test_update_is_member_mean_and_preserves_sum():
    rng = np.random.default_rng(6)
    X = rng.normal(size=(200, 5))
    lab = rng.integers(0, 9, size=200)
    lab[lab == 4] = 5                      # cluster 4 empty
    prev = rng.normal(size=(9, 5))
    C = svoo.update_centroids(X, lab, prev)
    sizes = np.bincount(lab, minlength=9)
    np.testing.assert_allclose((C * sizes[:, None]).sum(0), X.sum(0), atol=1e-11)
    assert np.array_equal(C[4], prev[4])
    for j in range(9):
        if sizes[j]:
            # the mean is the unique minimiser of sum ||x - c||^2: gradient zero
            np.testing.assert_allclose((X[lab == j] - C[j]).sum(0), 0, atol=1e-11)


# ---------------------------------------------------------------- permutation
@pytest.mark.parametrize("K", [1, 7, 100])
def test_counting_sort_matches_stable_argsort(K):
    lab = np.random.default_rng(K).integers(0, K, size=5000)
    lab[lab == (K // 2)] = 0 if K > 1 else lab[lab == 0]
    perm, offs = svoo.counting_sort(lab, K)
    assert np.array_equal(perm, np.argsort(lab, kind="stable"))
    assert np.array_equal(offs, np.concatenate([[0], np.cumsum(np.bincount(lab, minlength=K))]))
    assert np.array_equal(np.sort(perm), np.arange(len(lab)))


# ---------------------------------------------------------------- selection
def test_recall_count_golden():
    for case in GOLD["recall_count"]:
        assert svoo.recall_count(case["p"], case["tau"]) == case["count"], case["cite"]


def test_recall_through_select_blocks():
    """SPEC row [0.5,0.3,0.1,0.1] realised as softmax(Abar/sqrt(d)) with C_k = I."""
    p = np.array([0.5, 0.3, 0.1, 0.1])
    Cq = (2.0 * np.log(p))[None, :]       # d = 4 -> sqrt(d) = 2
    r = svoo.select_blocks(Cq, np.eye(4), [5], [1, 1, 1, 1], 1.0, 0.8, 0.1, svoo.RULE_DENSITY)
    assert r.c[0] == 2 and r.n_rec == 2


def test_rho_rule_golden():
    rules = {"as_written": svoo.RULE_AS_WRITTEN, "density": svoo.RULE_DENSITY}
    for case in GOLD["rho_rule"]:
        Kk = 10
        n = svoo.rule_count(round(case["recall"] * Kk), case["budget"], case["theta"],
                            rules[case["rule"]], Kk, Kk)
        assert n == round(case["rho"] * Kk), case["cite"]


def test_mask_golden():
    for case in GOLD["mask"]:
        row = np.array(case["row"])
        k = len(row)
        r = svoo.select_blocks(row[None, :], np.eye(k), [1], [1] * k, case["rho"], 0.95, 0.1,
                               svoo.RULE_FIXED)
        assert list(r.kept[0]) == case["kept"], case["cite"]


def test_n_from_ratio_exact_decimals():
    """R10: matches exact rational ceil(b*K) for every 3-decimal budget at K in {100, 500, 1024}."""
    from fractions import Fraction
    for Kk in (100, 500, 1024):
        for m in range(1, 1001):
            b = float(np.float32(m / 1000))
            exact = math.ceil(Fraction(m, 1000) * Kk)
            assert svoo.n_from_ratio(b, Kk) == min(max(exact, 1), Kk), (Kk, m)


def test_masks_nested_and_full_budget():
    rng = np.random.default_rng(8)
    Cq, Ck = rng.normal(size=(6, 8)), rng.normal(size=(30, 8))
    sk = np.ones(30, int)
    sk[[3, 17]] = 0
    prev = None
    for b in (0.05, 0.2, 0.5, 0.9, 1.0):
        r = svoo.select_blocks(Cq, Ck, np.ones(6), sk, b, 0.95, 0.1, svoo.RULE_FIXED)
        assert not np.isin(r.kept, [3, 17]).any()
        if prev is not None:
            for a in range(6):
                assert set(prev[a]) <= set(r.kept[a])
        prev = r.kept
    assert r.n_keep == 28


# ---------------------------------------------------------------- attention
def test_full_keep_equals_library_sdpa():
    rng = np.random.default_rng(9)
    for n in (8, 64, 256):
        Q, K, V = rng.normal(size=(3, n, 16))
        Lq = rng.integers(0, 3, n)
        Lk = rng.integers(0, 4, n)
        kept = np.tile(np.arange(4), (3, 1))
        O = svoo.sparse_attention(Q, K, V, Lq, Lk, kept)
        ref = torch.nn.functional.scaled_dot_product_attention(
            torch.from_numpy(Q)[None], torch.from_numpy(K)[None], torch.from_numpy(V)[None])[0]
        np.testing.assert_allclose(O, ref.numpy(), atol=1e-12)
        np.testing.assert_allclose(svoo.dense_attention(Q, K, V), ref.numpy(), atol=1e-12)


def test_singleton_blocks_pick_argmax_value():
    """S:385 / S:422: singleton blocks -> Abar = Q K^T; keeping 1 block gives v[argmax_j q.k_j]."""
    rng = np.random.default_rng(10)
    n = 40
    Q, K, V = rng.normal(size=(3, n, 8))
    ones = np.ones(n, int)
    r = svoo.select_blocks(Q, K, ones, ones, 1.0 / n, 0.95, 0.1, svoo.RULE_FIXED)
    assert r.n_keep == 1
    np.testing.assert_allclose(r.Abar, Q @ K.T, atol=1e-12)
    O = svoo.sparse_attention(Q, K, V, np.arange(n), np.arange(n), r.kept)
    np.testing.assert_allclose(O, V[(Q @ K.T).argmax(1)], atol=1e-12)


def test_bruteforce_n8_masked_softmax():
    rng = np.random.default_rng(11)
    Q, K, V = rng.normal(size=(3, 8, 4))
    Lq = np.array([0, 1, 0, 1, 1, 0, 0, 1])
    Lk = np.array([0, 1, 2, 3, 0, 1, 2, 3])
    kept = np.array([[0, 2], [1, 3]])
    O = svoo.sparse_attention(Q, K, V, Lq, Lk, kept)
    for i in range(8):
        allowed = [j for j in range(8) if Lk[j] in kept[Lq[i]]]
        w = [math.exp(sum(Q[i, t] * K[j, t] for t in range(4)) / 2.0) for j in allowed]
        o = [sum(w[m] * V[allowed[m], t] for m in range(len(allowed))) / sum(w) for t in range(4)]
        np.testing.assert_allclose(O[i], o, atol=1e-12)
        assert np.all(O[i] >= V[allowed].min(0) - 1e-12) and np.all(O[i] <= V[allowed].max(0) + 1e-12)


# ---------------------------------------------------------------- whole layer
def _toy(seed=0, N_scale=1):
    from synthetic import video_qkv
    w = video_qkv(4, 8, 8 * N_scale, 1, 32, seed=seed)
    f = lambda t: t[0, 0].double().numpy()
    return f(w.q), f(w.k), f(w.v)


def test_layer_full_budget_equals_dense():
    Q, K, V = _toy()
    r = svoo.coclust_sparse_attention_head(Q, K, V, 8, 12, 2, 3, 1.0, 0.95, 0.1, svoo.RULE_FIXED)
    np.testing.assert_allclose(r.O, svoo.dense_attention(Q, K, V), atol=1e-12)


def test_token_order_invariance():
    Q, K, V = _toy(seed=1)
    N = Q.shape[0]
    pi = np.random.default_rng(12).permutation(N)      # new position p holds old token pi[p]
    inv = np.argsort(pi)
    iq = svoo.sample_anchor_indices(N, 8, 5, 0, 0, 1, 0)
    ik = svoo.sample_anchor_indices(N, 12, 5, 0, 0, 1, 1)
    a = svoo.cocluster(Q, K, 8, 12, 2, init_q=iq, init_k=ik)
    b = svoo.cocluster(Q[pi], K[pi], 8, 12, 2, init_q=inv[iq], init_k=inv[ik])
    assert np.array_equal(a.Lq[pi], b.Lq) and np.array_equal(a.Lk[pi], b.Lk)
    np.testing.assert_allclose(a.Cq, b.Cq, atol=1e-12)
    sa = svoo.select_blocks(a.Cq, a.Ck, np.bincount(a.Lq, minlength=8), np.bincount(a.Lk, minlength=12),
                            0.3, 0.95, 0.1, svoo.RULE_DENSITY)
    Oa = svoo.sparse_attention(Q, K, V, a.Lq, a.Lk, sa.kept)
    Ob = svoo.sparse_attention(Q[pi], K[pi], V[pi], b.Lq, b.Lk, sa.kept)
    np.testing.assert_allclose(Oa[pi], Ob, atol=1e-12)


def test_assignment_halfstep_nonincreasing_and_optimal():
    """With the centroids held fixed, each assignment is optimal (no token improves by switching),
    hence the half-step objective cannot exceed that of the previous labels."""
    Q, K, _ = _toy(seed=2)
    res = svoo.cocluster(Q, K, 8, 12, 3, seed=1)
    for t in res.trace:
        X = K if t["side"] == "k" else Q
        r = svoo.assign_step(X, t["C_anchor"], t["C_self"])
        P = svoo.l2_normalize_rows(X @ t["C_anchor"].T)
        Pb = svoo.l2_normalize_rows(t["C_self"] @ t["C_anchor"].T)
        D = np.linalg.norm(P[:, None, :] - Pb[None, :, :], axis=2)
        assert np.all(D[np.arange(len(X)), r.labels] <= D.min(1) + 1e-12)


def test_toy_config_runs_fast():
    import time
    from synthetic import config_workload
    w = config_workload("toy")
    f = lambda t: t[0, 0].double().numpy()
    t0 = time.time()
    r = svoo.coclust_sparse_attention_head(f(w.q), f(w.k), f(w.v), 16, 16, 3, 0, 0.3, 0.95, 0.1,
                                           svoo.RULE_DENSITY)
    assert time.time() - t0 < 30
    assert r.sel.n_keep >= 1 and r.O.shape == (2048, 64)
    assert np.isfinite(r.O).all()


# ------------------------------------------------------------------ NEXT-4 selection variants
def _rand_select_inputs(seed, kq=12, kk=30, d=16):
    rng = np.random.default_rng(seed)
    Cq, Ck = rng.normal(size=(kq, d)), rng.normal(size=(kk, d))
    sq = rng.integers(0, 9, kq)
    sk = rng.integers(0, 9, kk)
    sq[0] = sk[0] = 3  # at least one nonempty block on each side
    return Cq, Ck, sq, sk


@pytest.mark.parametrize("seed", range(4))
def test_size_weighted_equal_sizes_reduces_to_base(seed):
    """log|K_c| is a constant when all key blocks have the same size: softmax and ranking are
    shift invariant, so the weighted selection equals the base reading (R9)."""
    Cq, Ck, sq, _ = _rand_select_inputs(seed)
    sk = np.full(Ck.shape[0], 5)
    for rule in (svoo.RULE_DENSITY, svoo.RULE_FIXED):
        a = svoo.select_blocks(Cq, Ck, sq, sk, 0.2, 0.9, 0.1, rule)
        b = svoo.select_blocks(Cq, Ck, sq, sk, 0.2, 0.9, 0.1, rule, size_weighted=True)
        assert a.n_keep == b.n_keep and np.array_equal(a.c, b.c)
        assert np.array_equal(a.kept, b.kept)


def test_size_weighted_closed_form_masses():
    """Two key blocks with the same centroid logit but sizes 1 and 9: the weighted masses are
    1/10 and 9/10 (p_c = |K_c| e^{z_c} / sum |K| e^z), so tau = 0.85 is covered by the large
    block alone (c = 1) while the unweighted masses 1/2, 1/2 need both (c = 2)."""
    Cq = np.array([[1.0, 0.0]])
    Ck = np.array([[1.0, 0.0], [1.0, 0.0], [-50.0, 0.0]])
    sq, sk = np.array([4]), np.array([1, 9, 2])
    w = svoo.select_blocks(Cq, Ck, sq, sk, 1.0, 0.85, 0.1, svoo.RULE_FIXED, size_weighted=True)
    u = svoo.select_blocks(Cq, Ck, sq, sk, 1.0, 0.85, 0.1, svoo.RULE_FIXED)
    assert w.c[0] == 1 and u.c[0] == 2
    # the weighted order puts block 1 (size 9) first; the unweighted tie goes to index 0
    p_w = np.array([1.0, 9.0]) / 10.0
    assert p_w[1] >= 0.85 > p_w[0]
    z = Cq @ Ck.T / math.sqrt(2) + np.log(sk)
    assert np.argmax(z[0]) == 1


@pytest.mark.parametrize("seed", range(4))
def test_per_row_fixed_equals_shared(seed):
    """FIXED: every row keeps n_b blocks, so per-row counts equal the shared count."""
    Cq, Ck, sq, sk = _rand_select_inputs(seed)
    a = svoo.select_blocks(Cq, Ck, sq, sk, 0.3, 0.9, 0.1, svoo.RULE_FIXED)
    b = svoo.select_blocks(Cq, Ck, sq, sk, 0.3, 0.9, 0.1, svoo.RULE_FIXED, per_row=True)
    assert np.all(b.n_rows == a.n_keep)
    assert all(np.array_equal(a.kept[r], b.kept[r]) for r in range(len(sq)))


def test_per_row_hand_example():
    """Row 0 has one dominant key block (c_0 = 1), row 1 three equal ones (masses 1/3 each,
    tau = 0.9 -> c_1 = 3).  Budget 0.5 of 6 blocks -> n_b = 3, density rule with 1-b > theta ->
    min.  Shared (R11): n_rec = ceil(4/2) = 2 -> both rows keep 2.  Per row: 1 and 3."""
    Cq = np.array([[20.0, 0.0], [0.0, 20.0]])
    Ck = np.array([[20.0, 0.0], [0.0, 20.0], [0.0, 20.0], [0.0, 20.0], [0.0, 0.0], [0.0, 0.0]])
    sq, sk = np.array([5, 5]), np.ones(6, int)
    sh = svoo.select_blocks(Cq, Ck, sq, sk, 0.5, 0.9, 0.1, svoo.RULE_DENSITY)
    pr = svoo.select_blocks(Cq, Ck, sq, sk, 0.5, 0.9, 0.1, svoo.RULE_DENSITY, per_row=True)
    assert list(sh.c) == [1, 3] and sh.n_rec == 2 and sh.n_keep == 2
    assert sh.kept.tolist() == [[0, 1], [1, 2]]
    assert pr.n_rows.tolist() == [1, 3]
    assert [k.tolist() for k in pr.kept] == [[0], [1, 2, 3]]


def test_per_row_empty_query_block_keeps_shared_n():
    Cq, Ck, sq, sk = _rand_select_inputs(7)
    sq[3] = 0
    pr = svoo.select_blocks(Cq, Ck, sq, sk, 0.2, 0.9, 0.1, svoo.RULE_DENSITY, per_row=True)
    assert pr.n_rows[3] == pr.n_keep
    for a in range(len(sq)):
        if sq[a] > 0:
            assert pr.n_rows[a] == svoo.rule_count(int(pr.c[a]), 0.2, 0.1, svoo.RULE_DENSITY, len(sk),
                                                   int((sk > 0).sum()))


# ------------------------------------------------------------------ NEXT-2 k-means baseline + recall
def _blobs(n_per, centers, seed, sd=0.3):
    rng = np.random.default_rng(seed)
    X = np.concatenate([c + sd * rng.normal(size=(n_per, len(c))) for c in centers])
    return X, np.repeat(np.arange(len(centers)), n_per)


def test_kmeans_matches_sklearn_lloyd():
    """Independent k-means (the "w/o On" partitioning) = textbook Lloyd: sklearn's KMeans
    (algorithm="lloyd", the same initial centroids, n_init=1) reaches the same centroids."""
    from sklearn.cluster import KMeans
    rng = np.random.default_rng(3)
    centers = rng.normal(size=(6, 8)) * 3
    X, _ = _blobs(40, centers, 4, sd=1.0)
    init = np.array([0, 45, 90, 130, 170, 230])     # one token per blob: no empty cluster
    for iters in (1, 2, 5):
        L, C, _ = svoo.kmeans(X, 6, iters, init=init)
        km = KMeans(n_clusters=6, init=X[init], n_init=1, max_iter=iters, algorithm="lloyd", tol=0.0).fit(X)
        assert np.allclose(C, km.cluster_centers_, atol=1e-10)
        # our labels are those of the last assignment (R13); sklearn's of its final E-step
        assert np.array_equal(svoo.kmeans_step(X, C).labels, km.labels_)


def test_kmeans_objective_nonincreasing_and_recovers_blobs():
    rng = np.random.default_rng(5)
    centers = rng.normal(size=(5, 16)) * 4
    X, truth = _blobs(50, centers, 6)
    L, C, tr = svoo.kmeans(X, 5, 6, seed=1)
    J = [t["J"] for t in tr]
    assert all(J[i + 1] <= J[i] + 1e-9 for i in range(len(J) - 1))
    # well-separated blobs seeded one token per blob: the partition is the truth up to relabelling
    L2, _, _ = svoo.kmeans(X, 5, 3, init=np.arange(5) * 50 + 7)
    assert len({(a, b) for a, b in zip(L2, truth)}) == 5 and len(np.unique(L2)) == 5


def test_reference_pairs_minimal_prefix_bruteforce():
    rng = np.random.default_rng(7)
    S = rng.normal(size=(6, 6)) * 2
    A = np.exp(S - S.max(1, keepdims=True))
    A /= A.sum(1, keepdims=True)
    ref = svoo.reference_pairs(A, 0.5)
    assert A[ref].sum() >= 0.5 * A.sum() - 1e-12
    # minimality: dropping the smallest selected pair goes below the target, and every unselected
    # pair is no larger than every selected one
    assert A[ref].sum() - A[ref].min() < 0.5 * A.sum()
    assert A[~ref].max() <= A[ref].min()


def test_block_pair_recall_special_partitions():
    rng = np.random.default_rng(8)
    S = rng.normal(size=(12, 12))
    A = np.exp(S) / np.exp(S).sum(1, keepdims=True)
    ref = svoo.reference_pairs(A, 0.5)
    n = int(ref.sum())
    ident = np.arange(12)
    cnt = svoo.block_pair_counts(ref, ident, ident, 12, 12)
    assert np.array_equal(cnt, ref.astype(np.int64))
    assert svoo.pairs_to_cover(cnt) == n and svoo.block_pair_recall(cnt, n) == 1.0
    assert svoo.block_pair_recall(cnt, n - 1) == (n - 1) / n
    one = np.zeros(12, int)
    cnt1 = svoo.block_pair_counts(ref, one, one, 1, 1)
    assert cnt1[0, 0] == n and svoo.block_pair_recall(cnt1, 1) == 1.0 and svoo.pairs_to_cover(cnt1) == 1


# ------------------------------------------------------------------ NEXT-3 offline profiler
def test_density_closed_forms():
    n = 40
    U = np.full((3, n), 1.0 / n)                      # uniform rows: ceil(tau n) entries
    for tau in (0.95, 0.5, 0.9, 1.0):
        d, c = svoo.attention_density(U, tau)
        assert np.all(c == math.ceil(tau * n - 1e-9)) and d == math.ceil(tau * n - 1e-9) / n
    E = np.eye(n)                                     # one-hot rows: a single entry
    d, c = svoo.attention_density(E, 0.95)
    assert np.all(c == 1) and d == 1.0 / n
    r = 0.7                                           # geometric row p_j ~ r^j (any column order)
    g = r ** np.arange(n)
    g /= g.sum()
    perm = np.random.default_rng(0).permutation(n)
    d, c = svoo.attention_density(g[perm][None], 0.95)
    m = next(m for m in range(1, n + 1) if (1 - r ** m) / (1 - r ** n) >= 0.95)
    assert c[0] == m


def test_density_minimal_subset_bruteforce():
    """The sorted prefix is the minimal subset reaching tau: check against all subsets (n = 7)."""
    rng = np.random.default_rng(2)
    for _ in range(5):
        p = rng.dirichlet(np.ones(7) * 0.5)
        best = min(len(sub) for k in range(1, 8) for sub in itertools.combinations(range(7), k)
                   if p[list(sub)].sum() >= 0.8 - 1e-12)
        assert svoo.attention_density(p[None], 0.8)[1][0] == best


def test_density_qk_and_schedule():
    rng = np.random.default_rng(4)
    Q, K = rng.normal(size=(30, 16)), rng.normal(size=(30, 16))
    d, c = svoo.attention_density_qk(Q, K, 0.95)
    S = Q @ K.T / 4.0
    A = np.exp(S - S.max(1, keepdims=True))
    A /= A.sum(1, keepdims=True)
    assert d == svoo.attention_density(A, 0.95)[0] and 0 < d <= 1
    from scipy.stats import norm
    assert abs(svoo.Z_95 - norm.ppf(0.95)) < 1e-12
    dens = np.array([[[0.1, 0.5]], [[0.3, 0.7]]])     # m = 2 inputs, 1 layer, 2 heads
    sch = svoo.sparsity_schedule(dens)
    assert np.allclose(sch["mu"], [[0.2, 0.6]]) and np.allclose(sch["sigma"], [[0.1, 0.1]])
    assert np.allclose(sch["d_hat"], [[0.2 + 0.1 * norm.ppf(0.95), min(1.0, 0.6 + 0.1 * norm.ppf(0.95))]])
    assert np.allclose(sch["s"], 1 - sch["d_hat"])


def test_density_golden_spec_examples():
    """uniform 10-wide rows at tau = 0.8 -> 0.8; one-hot rows -> 1/n;
    row [0.5, 0.3, 0.1, 0.1] at tau = 0.8 -> 0.5."""
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))["recall_count"]
    for ex in g:
        p = np.asarray(ex["p"], np.float64)
        d, c = svoo.attention_density(p[None], ex["tau"])
        assert c[0] == ex["count"] and d == ex["count"] / len(p)
    assert svoo.attention_density(np.eye(7), 0.3)[0] == 1 / 7


def test_recall_counts_equal_row_density_of_softmaxed_abar():
    """SURVEY 4.1 invariant: Recall's c_a (R9) is the attention-density prefix of the row
    softmax(Abar_a / sqrt(d)) over the nonempty key blocks."""
    Cq, Ck, sq, sk = _rand_select_inputs(11, kq=10, kk=40, d=16)
    sel = svoo.select_blocks(Cq, Ck, sq, sk, 0.3, 0.9, 0.1, svoo.RULE_DENSITY, d_head=16)
    ne = sk > 0
    A = (Cq @ Ck.T)[:, ne] / 4.0
    P = np.exp(A - A.max(1, keepdims=True))
    P /= P.sum(1, keepdims=True)
    _, c = svoo.attention_density(P, 0.9)
    for a in range(len(sq)):
        if sq[a] > 0:
            assert sel.c[a] == c[a]


def test_sparse_error_monotone_in_keep_ratio():
    """SPEC invariant (nested masks): the median row error of the sparse output against
    dense attention does not grow as rho grows (FIXED rule), and vanishes at rho = 1."""
    rng = np.random.default_rng(12)
    N, d = 256, 16
    centers = rng.normal(size=(8, d)) * 2
    lab = rng.integers(0, 8, N)
    Q = centers[lab] + 0.7 * rng.normal(size=(N, d))
    K = centers[lab] + 0.7 * rng.normal(size=(N, d))
    V = rng.normal(size=(N, d))
    dense = svoo.dense_attention(Q, K, V)
    errs = []
    for rho in (0.1, 0.25, 0.5, 0.75, 1.0):
        r = svoo.coclust_sparse_attention_head(Q, K, V, 8, 16, 2, 0, rho, 0.95, 0.1, svoo.RULE_FIXED)
        errs.append(float(np.median(np.linalg.norm(r.O - dense, axis=1))))
    assert all(b <= a + 1e-12 for a, b in zip(errs, errs[1:])), errs
    assert errs[-1] < 1e-12
