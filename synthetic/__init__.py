"""Seeded synthetic workloads shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the method's arithmetic (no clustering, selection or attention):
it only draws inputs.  Recipe:

* tokens sit on the latent grid (T, Hs, Ws), Wan flatten order i = (t*Hs + y)*Ws + x;
* per (layer, head) stream seed = base ^ (layer*1000 + head);
* 64 region seeds uniform in the normalised (t/T, y/Hs, x/Ws) cube, time axis weighted 0.5;
  region r(i) = nearest seed (Voronoi cell) -> spatially coherent blobs of uneven size;
* region centres c_r ~ N(0, I_d); Q_i = c_r(i) + 0.8 eps, K_i = c_r(i) + 0.8 eps', V ~ N(0, 1);
* everything is rounded to bf16 once; both the oracle and the CUDA path consume those values.

Per-layer budgets ("synthetic offline profile", P:1186-1189 formula only):
  base_l ~ U(0.03, 0.40); mu = base_l + 0.02 N(0,1); sigma ~ U(0.005, 0.03);
  d_hat = min(1, mu + 1.6449 sigma); layer 0 -> 1.0 (layer warm-up).
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

# (T, Hs, Ws, H, d) of the BASELINE.json configs
CONFIGS = {
    "toy": dict(T=8, Hs=16, Ws=16, H=1, d=64, kq=16, kk=16, iters=3, budget=0.3),
    "wan1.3b_480p": dict(T=21, Hs=30, Ws=52, H=12, d=128, kq=100, kk=500, iters=2, budget=None),
    "wan14b_720p": dict(T=21, Hs=45, Ws=80, H=40, d=128, kq=100, kk=500, iters=2, budget=0.2),
    "hunyuan_720p": dict(T=33, Hs=45, Ws=80, H=24, d=128, kq=100, kk=500, iters=2, budget=0.2),
}


@dataclass
class Workload:
    q: torch.Tensor   # bf16 [B, H, N, d]
    k: torch.Tensor
    v: torch.Tensor
    regions: torch.Tensor  # int64 [H, N] (ground-truth blob id, diagnostics only)


def _regions(T, Hs, Ws, n_regions, gen, device):
    t = torch.arange(T, device=device, dtype=torch.float32) / T
    y = torch.arange(Hs, device=device, dtype=torch.float32) / Hs
    x = torch.arange(Ws, device=device, dtype=torch.float32) / Ws
    tt, yy, xx = torch.meshgrid(t, y, x, indexing="ij")
    coords = torch.stack([0.5 * tt.reshape(-1), yy.reshape(-1), xx.reshape(-1)], 1)   # [N, 3]
    seeds = torch.rand(n_regions, 3, generator=gen, device=device)
    seeds[:, 0] *= 0.5
    dist = torch.cdist(coords, seeds)
    return dist.argmin(1)


def video_qkv(T: int, Hs: int, Ws: int, H: int, d: int, *, seed: int = 0, layer: int = 0,
              B: int = 1, n_regions: int = 64, noise: float = 0.8, device="cpu",
              layout: str = "bhnd") -> Workload:
    """Q/K/V for one attention layer, bf16.  layout 'bhnd' -> [B,H,N,d] contiguous;
    'bnhd' -> a [B,N,H,d] buffer returned as a [B,H,N,d] strided view."""
    N = T * Hs * Ws
    dev = torch.device(device)
    qs, ks, vs, rs = [], [], [], []
    for b in range(B):
        for h in range(H):
            gen = torch.Generator(device=dev)
            gen.manual_seed((seed ^ (layer * 1000 + h + 7919 * b)) & 0x7FFFFFFFFFFFFFFF)
            r = _regions(T, Hs, Ws, n_regions, gen, dev)
            cent = torch.randn(n_regions, d, generator=gen, device=dev)
            qs.append(cent[r] + noise * torch.randn(N, d, generator=gen, device=dev))
            ks.append(cent[r] + noise * torch.randn(N, d, generator=gen, device=dev))
            vs.append(torch.randn(N, d, generator=gen, device=dev))
            rs.append(r)
    def pack(lst):
        t = torch.stack(lst).reshape(B, H, N, d).to(torch.bfloat16)
        if layout == "bnhd":
            t = t.permute(0, 2, 1, 3).contiguous().permute(0, 2, 1, 3)
        return t
    return Workload(pack(qs), pack(ks), pack(vs), torch.stack(rs))


def random_qkv(B: int, H: int, N: int, d: int, *, seed: int = 0, scale: float = 1.0,
               device="cpu") -> Workload:
    """Unstructured N(0, scale^2) Q/K and N(0,1) V (edge-case tests)."""
    gen = torch.Generator(device=torch.device(device))
    gen.manual_seed(seed)
    q = (scale * torch.randn(B, H, N, d, generator=gen, device=device)).to(torch.bfloat16)
    k = (scale * torch.randn(B, H, N, d, generator=gen, device=device)).to(torch.bfloat16)
    v = torch.randn(B, H, N, d, generator=gen, device=device).to(torch.bfloat16)
    return Workload(q, k, v, torch.zeros(H, N, dtype=torch.long))


def config_workload(name: str, *, seed: int = 0, layer: int = 0, device="cpu", H: int | None = None,
                    layout: str = "bhnd") -> Workload:
    c = CONFIGS[name]
    return video_qkv(c["T"], c["Hs"], c["Ws"], c["H"] if H is None else H, c["d"], seed=seed,
                     layer=layer, device=device, layout=layout)


def synthetic_profile(n_layers: int, H: int, *, seed: int = 0) -> torch.Tensor:
    """Per-(layer, head) keep budgets d_hat in (0, 1], float32 [L, H]."""
    gen = torch.Generator()
    gen.manual_seed(seed + 12345)
    base = 0.03 + 0.37 * torch.rand(n_layers, 1, generator=gen, dtype=torch.float64)
    mu = base + 0.02 * torch.randn(n_layers, H, generator=gen, dtype=torch.float64)
    sigma = 0.005 + 0.025 * torch.rand(n_layers, H, generator=gen, dtype=torch.float64)
    dhat = (mu + 1.6449 * sigma).clamp(1e-3, 1.0)
    dhat[0] = 1.0
    return dhat.to(torch.float32)


def random_labels(BH: int, N: int, K: int, *, seed: int = 0, empty: tuple = ()) -> torch.Tensor:
    """Labels for teacher-forced permute/update tests; clusters listed in `empty` are left empty."""
    gen = torch.Generator()
    gen.manual_seed(seed)
    lab = torch.randint(0, K, (BH, N), generator=gen, dtype=torch.int64)
    for c in empty:
        lab[lab == c] = (c + 1) % K if (c + 1) % K not in empty else 0
    return lab.to(torch.int32)
