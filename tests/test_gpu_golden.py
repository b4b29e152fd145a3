"""The hand-derived golden examples (tests/golden/alg1_examples.json) run through the C ABI: the
2-D vectors are zero-padded to d = 64 (no dot product changes), so the CUDA path must reproduce
the labels, centroids, selection counts and kept lists derived by hand from the paper — a
misreading shared by the oracle and the kernels would fail here.  Plus the defined result for a
caller-supplied kept row with no allowed key."""
import json
import os

import numpy as np
import pytest
import torch

from oracle import svoo

pytestmark = pytest.mark.gpu

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "alg1_examples.json")))
D = 64


@pytest.fixture(scope="module")
def pb():
    from paper_2603_18636_b200 import build
    build.build()
    import paper_2603_18636_b200 as m
    m.lib()
    return m


def pad(rows, dtype=torch.bfloat16):
    a = np.zeros((len(rows), D))
    a[:, :2] = np.asarray(rows, np.float64)
    return torch.from_numpy(a).to(dtype)


def idx(v):
    return torch.tensor(v, dtype=torch.int32)[None, None].cuda()


@pytest.mark.parametrize("iters", [1, 2])
def test_golden_alg1_two_iterations(pb, iters):
    ex = G["alg1_two_iterations"]
    exp = ex[f"iters_{iters}"]
    Q = pad(ex["Q"])[None, None].cuda()
    # N = 6 on both sides: two extra keys, copies of k1 and k4 (same cluster, so the member means
    # and hence every later half-step are unchanged)
    K = pad(ex["K"] + [ex["K"][0], ex["K"][3]])[None, None].cuda()
    st = pb.coclust_assign(Q, K, ex["kq"], ex["kk"], iters, init_q=idx(ex["init_q"]), init_k=idx(ex["init_k"]))
    torch.cuda.synchronize()
    assert st["lk"][0, 0].tolist() == exp["Lk"] + [exp["Lk"][0], exp["Lk"][3]]
    assert st["lq"][0, 0].tolist() == exp["Lq"]
    np.testing.assert_allclose(st["cq"][0, 0, :, :2].cpu().numpy(), exp["Cq"], rtol=1e-6, atol=1e-7)
    np.testing.assert_allclose(st["ck"][0, 0, :, :2].cpu().numpy(), exp["Ck"], rtol=1e-6, atol=1e-7)
    assert float(st["cq"][0, 0, :, 2:].abs().max()) == 0.0


def test_golden_fig3_coupling(pb):
    ex = G["fig3_coupling"]
    Q = pad(ex["Q"] * 2)[None, None].cuda()                     # N = 4: [q1, q2, q1, q2]
    K = pad(ex["K"])[None, None].cuda()
    parts = []
    for case in ex["anchored"]:
        st = pb.coclust_assign(Q, K, ex["kq"], ex["kk"], ex["iters"], init_q=idx(case["init_q"]),
                               init_k=idx(ex["init_k"]))
        torch.cuda.synchronize()
        lk = st["lk"][0, 0].tolist()
        assert lk == case["Lk"], ex["cite"]
        parts.append(lk)
    assert parts[0] != parts[1]


def test_golden_gap_example_label(pb):
    ex = G["gap_closed_form"]
    X = pad(ex["X"] + ex["X"])[None, None].cuda()
    lab = pb.coclust_assign_step(X, pad(ex["C_anchor"], torch.float32)[None, None].cuda(),
                                 pad(ex["C_self"], torch.float32)[None, None].cuda())
    assert lab[0, 0].tolist() == [ex["label"]] * 2


@pytest.mark.parametrize("budget,n_keep", [(0.5, 2), (0.95, 4)])
def test_golden_n_rec_and_density_branch(pb, budget, n_keep):
    """n_rec = ceil(3 / 2) = 2 over the NONEMPTY query blocks; DENSITY at b = 0.5 takes min
    (2), at b = 0.95 the max branch (n_b = 4 = all nonempty key blocks).  With d = 64 the softmax
    temperature is 1/8 instead of 1/sqrt2: the masses are still (1, ~0) and (1/2, 1/2) rows."""
    ex = G["n_rec"]
    cq = pad(ex["Cq"], torch.float32)[None, None].cuda()
    ck = pad(ex["Ck"], torch.float32)[None, None].cuda()
    oq = torch.tensor(np.concatenate([[0], np.cumsum(ex["sizes_q"])]), dtype=torch.int32)[None, None].cuda()
    ok = torch.tensor(np.concatenate([[0], np.cumsum(ex["sizes_k"])]), dtype=torch.int32)[None, None].cuda()
    n, kept = pb.block_select(cq, ck, oq, ok, torch.tensor([budget]).cuda(), ex["tau"], ex["theta"],
                              pb.RULE_DENSITY)
    torch.cuda.synchronize()
    assert int(n[0, 0]) == n_keep
    if n_keep == 2:
        assert kept[0, 0, :2, :2].tolist() == ex["kept_rows"]
    else:
        assert kept[0, 0, :2, :4].tolist() == [[0, 1, 2, 3]] * 2


def test_empty_allowed_key_set_gives_zero_rows(pb):
    """A caller-supplied kept row listing only empty key clusters (S:419's contract violation,
    which block_select never produces) has a defined result: o_i = 0 for that query block, and
    every other block is unaffected (checked against the oracle)."""
    from synthetic import random_qkv
    N, d, kq, kk = 1000, 128, 4, 6
    w = random_qkv(1, 1, N, d, seed=11)
    rng = np.random.default_rng(0)
    Lq = rng.integers(0, kq, N)
    Lk = rng.integers(0, kk, N)
    Lk[Lk == 5] = 4                                   # key cluster 5 is empty
    Lk[Lk == 2] = 1                                   # and so is 2
    pq, oq = svoo.counting_sort(Lq, kq)
    pk, ok = svoo.counting_sort(Lk, kk)
    kept = np.full((kq, kk), -1, np.int64)
    kept[0, :2] = [2, 5]                               # row 0: only empty clusters
    kept[1, :2] = [0, 1]
    kept[2, :2] = [3, 4]
    kept[3, :2] = [0, 4]
    t = lambda a: torch.from_numpy(np.asarray(a).astype(np.int32))[None, None].cuda()
    O = pb.block_sparse_attn(w.q.cuda(), w.k.cuda(), w.v.cuda(), t(pq), t(oq), t(pk), t(ok),
                             torch.full((1, 1), 2, dtype=torch.int32).cuda(), t(kept))
    torch.cuda.synchronize()
    O = O[0, 0].float().cpu().double().numpy()
    assert np.all(O[Lq == 0] == 0.0)
    rest = Lq != 0
    f = lambda x: x[0, 0].double().numpy()
    rows_ref = svoo.sparse_attention(f(w.q)[rest], f(w.k), f(w.v), Lq[rest], Lk, kept[:, :2])
    err = np.abs(O[rest] - rows_ref)
    assert err.max() <= 2e-2 and err.mean() <= 5e-3
