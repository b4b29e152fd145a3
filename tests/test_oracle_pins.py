"""Hand-derived pins for the oracle's Algorithm 1 wiring and selection count rules
(tests/golden/alg1_examples.json).  Each expected value there is derived by hand from the paper
(the derivation is stored beside it), so a misreading in oracle/svoo.py — a wrong centroid
generation in a half-step, swapped anchor/self roles, pre-update centroids returned, a floor in
n_rec, K_q instead of K_q', the wrong DENSITY branch, the gap on squared distances, a swapped R4
stream — fails here.  CPU only."""
import json
import os

import numpy as np
import pytest

from oracle import svoo

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "alg1_examples.json")))


def _arr(x):
    return np.asarray(x, np.float64)


# ---------------------------------------------------------------- Fig. 3
def test_fig3_key_partition_is_query_dependent():
    ex = G["fig3_coupling"]
    parts = []
    for case in ex["anchored"]:
        r = svoo.cocluster(_arr(ex["Q"]), _arr(ex["K"]), ex["kq"], ex["kk"], ex["iters"],
                           init_q=np.array(case["init_q"]), init_k=np.array(ex["init_k"]))
        assert r.Lk.tolist() == case["Lk"], ex["cite"]
        parts.append({frozenset(np.nonzero(r.Lk == c)[0].tolist()) for c in range(ex["kk"])})
    # the paper's statement: the two anchors induce different key groupings
    assert parts[0] != parts[1]
    assert parts[0] == {frozenset({0, 1}), frozenset({2, 3})}
    assert parts[1] == {frozenset({0, 3}), frozenset({1, 2})}


# ---------------------------------------------------------------- Alg. 1 wiring
@pytest.mark.parametrize("iters", [1, 2])
def test_alg1_hand_example(iters):
    ex = G["alg1_two_iterations"]
    exp = ex[f"iters_{iters}"]
    r = svoo.cocluster(_arr(ex["Q"]), _arr(ex["K"]), ex["kq"], ex["kk"], iters,
                       init_q=np.array(ex["init_q"]), init_k=np.array(ex["init_k"]))
    assert r.Lk.tolist() == exp["Lk"], "Step A (anchors C_q^(i-1), self C_k^(i-1))"
    assert r.Lq.tolist() == exp["Lq"], "Step B (anchors C_k^(i), self C_q^(i-1))"
    np.testing.assert_allclose(r.Ck, exp["Ck"], atol=1e-15, err_msg="R13: post-update C_k")
    np.testing.assert_allclose(r.Cq, exp["Cq"], atol=1e-15, err_msg="R13: post-update C_q")


def test_alg1_first_halfsteps_in_trace():
    """The instrumentation records, per half-step, what the GPU parity tests teacher-force: the
    hand example's first Step A and Step B with their anchor/self generations."""
    ex = G["alg1_two_iterations"]
    r = svoo.cocluster(_arr(ex["Q"]), _arr(ex["K"]), 2, 2, 1, init_q=np.array(ex["init_q"]),
                       init_k=np.array(ex["init_k"]))
    ta, tb = r.trace
    np.testing.assert_array_equal(ta["C_anchor"], np.eye(2))            # C_q^(0)
    np.testing.assert_array_equal(ta["C_self"], [[1, 1], [1, -1]])      # C_k^(0)
    np.testing.assert_array_equal(tb["C_anchor"], [[0, 1], [0, -1]])    # C_k^(1)
    np.testing.assert_array_equal(tb["C_self"], np.eye(2))              # C_q^(0)
    assert ta["labels"].tolist() == [0, 1, 1, 0] and tb["labels"].tolist() == [0, 1, 1, 0, 0, 1]


def _member_means(X, L, k):
    out = {}
    for j in range(k):
        rows = [X[i] for i in range(len(L)) if L[i] == j]
        if rows:
            out[j] = [sum(r[t] for r in rows) / len(rows) for t in range(X.shape[1])]
    return out


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_returned_centroids_are_member_means_of_returned_labels(seed):
    """R13: C_q, C_k returned by Alg. 1 are the means of the returned L_q, L_k; every
    empty cluster's row is one of the input tokens' previous centroid chain (here: checked to be
    an initial anchor row if the cluster was empty from the first update on)."""
    rng = np.random.default_rng(seed)
    Q, K = rng.normal(size=(60, 5)), rng.normal(size=(60, 5))
    r = svoo.cocluster(Q, K, 4, 7, 2, seed=seed)
    for X, L, C, k in ((Q, r.Lq, r.Cq, 4), (K, r.Lk, r.Ck, 7)):
        for j, m in _member_means(X, L, k).items():
            np.testing.assert_allclose(C[j], m, atol=1e-12)


# ---------------------------------------------------------------- gap
def test_gap_closed_form_unsquared():
    ex = G["gap_closed_form"]
    r = svoo.assign_step(_arr(ex["X"]), _arr(ex["C_anchor"]), _arr(ex["C_self"]))
    assert r.labels.tolist() == [ex["label"]]
    assert abs(r.gap[0] - ex["gap"]) < 1e-12, ex["why"]
    assert abs(r.dist_best[0] - ex["dist_best"]) < 1e-12


# ---------------------------------------------------------------- n_rec, DENSITY
def test_n_rec_ceil_over_nonempty_query_blocks():
    ex = G["n_rec"]
    r = svoo.select_blocks(_arr(ex["Cq"]), _arr(ex["Ck"]), ex["sizes_q"], ex["sizes_k"], ex["budget"],
                           ex["tau"], ex["theta"], svoo.RULE_DENSITY)
    assert r.c.tolist() == ex["c"], ex["why"]
    assert r.n_rec == ex["n_rec"] and r.n_keep == ex["n_keep"]
    assert r.kept[:2].tolist() == ex["kept_rows"]


def test_density_rule_branches():
    for case in G["density_branch"]["cases"]:
        n = svoo.rule_count(case["n_rec"], case["budget"], case["theta"], svoo.RULE_DENSITY,
                            case["Kk"], case.get("Kk_ne", case["Kk"]))
        assert n == case["n"], case["why"]


def test_density_max_branch_through_select_blocks():
    """b = 0.95 > 1 - theta: the max branch keeps every nonempty key block of the n_rec example."""
    ex = G["n_rec"]
    r = svoo.select_blocks(_arr(ex["Cq"]), _arr(ex["Ck"]), ex["sizes_q"], ex["sizes_k"], 0.95,
                           ex["tau"], 0.1, svoo.RULE_DENSITY)
    assert r.n_rec == 2 and r.n_keep == 4


# ---------------------------------------------------------------- R4 sampler literals
def test_r4_stream_seed_literals():
    for c in G["r4_literal"]["stream_seeds"]:
        assert svoo.sample_seed(c["seed"], c["b"], c["h"], c["H"], c["side"]) == int(c["stream"]), c["why"]


def test_r4_floyd_draw_literals():
    for c in G["r4_literal"]["draws"]:
        idx = svoo.sample_anchor_indices(c["N"], c["K"], c["seed"], c["b"], c["h"], c["H"], c["side"])
        assert idx.tolist() == c["idx"], c["why"]


def test_splitmix64_seed0_published_sequence():
    outs = [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F, 0xF88BB8A8724C81EC]
    s = 0
    for o in outs:
        s, v = svoo.splitmix64_next(s)
        assert v == o


def test_empty_cluster_keeps_centroid_effective_k():
    """R5: an empty cluster keeps its previous centroid (it may attract tokens again
    later) and is excluded from selection while empty.  The reference SPEC's CPU program instead
    reseeds it from the farthest token before the next assignment; here the effective count at
    selection is K_k' < K_k.  Construction: two keys are identical and both drawn as initial key
    centroids, so the higher index loses every tie (R2) in the first Step A."""
    rng = np.random.default_rng(7)
    Q = rng.normal(size=(40, 4))
    K = rng.normal(size=(40, 4))
    K[11] = K[5]
    init_k = np.array([5, 11, 20, 30])
    init_q = np.array([0, 10, 20])
    r1 = svoo.cocluster(Q, K, 3, 4, 1, init_q=init_q, init_k=init_k)
    sizes_k = np.bincount(r1.Lk, minlength=4)
    assert sizes_k[1] == 0 and np.array_equal(r1.Ck[1], K[11])   # empty, centroid kept (R5)
    sizes_q = np.bincount(r1.Lq, minlength=3)
    sel = svoo.select_blocks(r1.Cq, r1.Ck, sizes_q, sizes_k, 1.0, 0.95, 0.1, svoo.RULE_FIXED)
    assert sel.n_keep == 3                          # clamped to K_k' = 3, not K_k = 4
    for a in range(3):
        assert 1 not in set(np.asarray(sel.kept[a]).tolist())
    # with more iterations the kept (stale) centroid is what the next Step A sees, not a reseed
    r3 = svoo.cocluster(Q, K, 3, 4, 3, init_q=init_q, init_k=init_k)
    assert np.array_equal(r3.trace[2]["C_self"][1], K[11])
