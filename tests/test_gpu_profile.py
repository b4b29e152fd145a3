"""NEXT-3 offline profiler: GPU attention density against the float64 oracle.

The GPU scores are fp32 (bf16 MMA) and the oracle's fp64, so a row whose cumulative mass crosses
tau within rounding of an element boundary may differ by one entry: per-row prefix sizes must
match for >= 99% of the rows and within 2 everywhere; densities within 1e-4.
"""
import numpy as np
import pytest
import torch

from oracle import svoo
from synthetic import random_qkv, video_qkv

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pb():
    from paper_2603_18636_b200 import build
    build.build()
    import paper_2603_18636_b200 as m
    m.lib()
    return m


def f64(t):
    return t.detach().float().cpu().double().numpy()


@pytest.mark.parametrize("d,T,Hs,Ws,tau", [(128, 4, 16, 24, 0.95), (64, 2, 20, 25, 0.9), (128, 3, 16, 43, 0.5)])
def test_density_matches_oracle(pb, d, T, Hs, Ws, tau):
    w = video_qkv(T, Hs, Ws, 2, d, seed=d + T)           # N = 1536 / 1000 / 2064 (ragged tiles)
    dens, cnt = pb.attention_density(w.q.cuda(), w.k.cuda(), tau=tau, counts=True)
    torch.cuda.synchronize()
    for h in range(2):
        d_ref, c_ref = svoo.attention_density_qk(f64(w.q[0, h]), f64(w.k[0, h]), tau)
        c = cnt[0, h].cpu().numpy()
        diff = np.abs(c - c_ref)
        assert diff.max() <= 2 and (diff == 0).mean() >= 0.99, (diff.max(), (diff == 0).mean())
        assert abs(dens[0, h].item() - d_ref) <= 1e-4


def test_density_uniform_and_peaked_rows(pb):
    """q = 0: every row uniform -> |S| = ceil(tau N) exactly (all elements share the final
    interval, so the interpolation is exact).  Large scale with q = k: the diagonal dominates."""
    N, d = 1000, 64
    w = random_qkv(1, 1, N, d, seed=1)
    q0 = torch.zeros_like(w.q)
    dens, cnt = pb.attention_density(q0.cuda(), w.k.cuda(), tau=0.95, counts=True)
    torch.cuda.synchronize()
    assert (cnt.cpu() == 950).all() and abs(dens.item() - 0.95) < 1e-12
    dens, cnt = pb.attention_density(w.k.cuda(), w.k.cuda(), tau=0.95, scale=4.0, counts=True)
    torch.cuda.synchronize()
    d_ref, c_ref = svoo.attention_density_qk(f64(w.k[0, 0]), f64(w.k[0, 0]), 0.95, scale=4.0)
    assert np.abs(cnt[0, 0].cpu().numpy() - c_ref).max() <= 1 and abs(dens.item() - d_ref) < 1e-5


def test_density_fullsize_properties_and_schedule(pb):
    """Wan2.1-14B 720p head shape (N = 75,600): counts in [1, N], density monotone in tau, sampled
    rows against the oracle; then the Gaussian fit of the schedule module against the oracle's."""
    from paper_2603_18636_b200 import profiler
    w = video_qkv(21, 45, 80, 1, 128, seed=5, device="cuda")
    d95, c95 = pb.attention_density(w.q, w.k, tau=0.95, counts=True)
    d50 = pb.attention_density(w.q, w.k, tau=0.5)
    torch.cuda.synchronize()
    c = c95[0, 0].cpu().numpy()
    N = c.shape[0]
    assert c.min() >= 1 and c.max() <= N and d50.item() < d95.item()
    rows = np.random.default_rng(0).choice(N, 24, replace=False)
    Q, K = f64(w.q[0, 0][rows]), f64(w.k[0, 0])
    S = Q @ K.T / np.sqrt(128)
    A = np.exp(S - S.max(1, keepdims=True))
    A /= A.sum(1, keepdims=True)
    _, c_ref = svoo.attention_density(A, 0.95)
    assert np.abs(c[rows] - c_ref).max() <= 2
    dens = np.random.default_rng(1).uniform(0.02, 0.4, size=(10, 3, 4))
    got, ref = profiler.fit_schedule(dens), svoo.sparsity_schedule(dens)
    for key in ("mu", "sigma", "d_hat", "s"):
        assert np.allclose(got[key], ref[key], rtol=0, atol=1e-15)
