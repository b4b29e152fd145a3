"""Offline layer-wise sparsity schedule.

The per-(layer, head) attention densities come from the library (`attention_density`, one
tensor-core pass set per layer and calibration input); this module only fits the univariate
Gaussian over the m calibration inputs and writes the schedule:

    d_hat = min(1, mu + z_alpha sigma)   (alpha = 0.95, maximum-likelihood sigma)
    s     = 1 - d_hat

d_hat is the per-head keep budget the DENSITY rule consumes (R8); the clamp to 1 is
reading R21.
"""
from __future__ import annotations

import json

import numpy as np

import paper_2603_18636_b200 as pb

Z_ALPHA_95 = 1.6448536269514722


def layer_densities(q, k, tau=0.95, scale=None, passes=0, ws=None):
    """Densities of one layer for one calibration input: float64 [H] (B = 1)."""
    return pb.attention_density(q, k, tau=tau, scale=scale, passes=passes, ws=ws)[0].cpu().numpy()


def fit_schedule(densities, z=Z_ALPHA_95):
    """densities [m, L, H] -> dict of [L, H] arrays mu, sigma, d_hat, s."""
    d = np.asarray(densities, dtype=np.float64)
    mu = d.mean(axis=0)
    sigma = d.std(axis=0)
    d_hat = np.minimum(mu + z * sigma, 1.0)
    return {"mu": mu, "sigma": sigma, "d_hat": d_hat, "s": 1.0 - d_hat}


def save_schedule(path, sched, meta=None):
    out = {k: np.asarray(v).tolist() for k, v in sched.items()}
    out["meta"] = meta or {}
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
