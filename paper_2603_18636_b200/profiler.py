"""Offline layer-wise sparsity schedule.

The per-(layer, head) attention densities come from the library (`attention_density`: tensor-core
QK^T passes and a per-row radix select on the GPU, one call per layer and calibration input); this
module collects them over a calibration set, fits the univariate Gaussian of each (layer, head)
over its m samples and derives the schedule:

    d_hat = min(1, mu + z_alpha sigma)   (maximum-likelihood sigma; alpha = 0.95)
    s     = 1 - d_hat

d_hat is the per-head keep budget the DENSITY rule consumes (R8); the clamp to 1 is
reading R21.  The schedule is written in the JSON document the reference SPEC fixes:
{"tau", "alpha", "entries": [{"layer", "head", "mean", "std", "d_hat", "sparsity", "samples"}]},
entries sorted by (layer, head).  Host-side arithmetic only (numpy, float64): nothing here is on the
attention hot path.
"""
from __future__ import annotations

import json
import math
from typing import Callable, Iterable

import numpy as np

Z_ALPHA_95 = 1.6448536269514722  # upper 0.95 quantile of N(0, 1)


def normal_quantile(p: float) -> float:
    """Inverse of the standard normal CDF for p in (0, 1): Acklam's rational approximation
    (relative error < 1.2e-9) refined by two Newton steps on Phi(x) = erfc(-x / sqrt 2) / 2, taken
    in the lower tail (p > 1/2 by symmetry: 1 - p is exact there), so the tails keep full
    relative precision."""
    if not 0.0 < p < 1.0:
        raise ValueError(f"quantile level must be in (0, 1), got {p}")
    if p > 0.5:
        return -normal_quantile(1.0 - p)
    a = (-3.969683028665376e+01, 2.209460984245205e+02, -2.759285104469687e+02,
         1.383577518672690e+02, -3.066479806614716e+01, 2.506628277459239e+00)
    b = (-5.447609879822406e+01, 1.615858368580409e+02, -1.556989798598866e+02,
         6.680131188771972e+01, -1.328068155288572e+01)
    c = (-7.784894002430293e-03, -3.223964580411365e-01, -2.400758277161838e+00,
         -2.549732539343734e+00, 4.374664141464968e+00, 2.938163982698783e+00)
    e = (7.784695709041462e-03, 3.224671290700398e-01, 2.445134137142996e+00, 3.754408661907416e+00)
    if p < 0.02425:
        q = math.sqrt(-2.0 * math.log(p))
        x = (((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) / \
            ((((e[0] * q + e[1]) * q + e[2]) * q + e[3]) * q + 1.0)
    else:
        q = p - 0.5
        r = q * q
        x = (((((a[0] * r + a[1]) * r + a[2]) * r + a[3]) * r + a[4]) * r + a[5]) * q / \
            (((((b[0] * r + b[1]) * r + b[2]) * r + b[3]) * r + b[4]) * r + 1.0)
    for _ in range(2):
        err = 0.5 * math.erfc(-x / math.sqrt(2.0)) - p
        x -= err * math.sqrt(2.0 * math.pi) * math.exp(0.5 * x * x)
    return x


def collect_densities(calibration: Iterable, n_layers: int, qk_of: Callable, tau: float = 0.95,
                      passes: int = 0, ws=None) -> np.ndarray:
    """Densities d^k_{l,h} of every calibration input k and layer l: float64 [m, L, H].

    `calibration` yields the inputs; `qk_of(x, layer)` returns that layer's (q, k) CUDA tensors
    [1, H, N, d] for input x.  Each (input, layer) is one `attention_density` call."""
    import paper_2603_18636_b200 as pb
    rows = []
    for x in calibration:
        per_layer = []
        for layer in range(n_layers):
            q, k = qk_of(x, layer)
            per_layer.append(pb.attention_density(q, k, tau=tau, passes=passes, ws=ws)[0].cpu().numpy())
        rows.append(per_layer)
    if not rows:
        raise ValueError("empty calibration set")
    return np.asarray(rows, dtype=np.float64)


def fit_schedule(densities, alpha: float = 0.95, tau: float = 0.95, z: float | None = None) -> dict:
    """densities [m, L, H] (m >= 1 samples per (layer, head), each in (0, 1]) -> schedule dict with
    [L, H] arrays mu, sigma (maximum likelihood, ddof 0), d_hat, s and the samples [L, H, m]."""
    d = np.asarray(densities, dtype=np.float64)
    if d.ndim != 3:
        raise ValueError(f"densities must be [m, L, H], got shape {d.shape}")
    if d.shape[0] == 0:
        raise ValueError("every (layer, head) needs at least one density sample")
    if not np.all(np.isfinite(d)) or d.min() <= 0.0 or d.max() > 1.0:
        raise ValueError("density samples must be finite and in (0, 1]")
    if not 0.5 <= alpha < 1.0:
        raise ValueError(f"alpha must be in [0.5, 1) (got {alpha})")
    if not 0.0 < tau <= 1.0:
        raise ValueError(f"tau must be in (0, 1] (got {tau})")
    zq = (Z_ALPHA_95 if alpha == 0.95 else normal_quantile(alpha)) if z is None else z
    mu = d.mean(axis=0)
    sigma = d.std(axis=0)
    d_hat = np.minimum(mu + zq * sigma, 1.0)
    return {"mu": mu, "sigma": sigma, "d_hat": d_hat, "s": 1.0 - d_hat, "samples": np.moveaxis(d, 0, -1),
            "alpha": float(alpha), "tau": float(tau), "z": float(zq)}


def to_spec(sched: dict, meta: dict | None = None) -> dict:
    """The schedule as the SPEC's JSON document, entries sorted by (layer, head)."""
    L, H = sched["d_hat"].shape
    entries = [{"layer": l, "head": h, "mean": float(sched["mu"][l, h]), "std": float(sched["sigma"][l, h]),
                "d_hat": float(sched["d_hat"][l, h]), "sparsity": float(sched["s"][l, h]),
                "samples": [float(v) for v in sched["samples"][l, h]]}
               for l in range(L) for h in range(H)]
    doc = {"tau": sched["tau"], "alpha": sched["alpha"], "entries": entries}
    if meta:
        doc["meta"] = meta
    return doc


def save_schedule(path: str, sched: dict, meta: dict | None = None) -> None:
    with open(path, "w") as f:
        json.dump(to_spec(sched, meta), f, indent=1)


def load_schedule(path_or_doc) -> dict:
    """Read a SPEC schedule document back: [L, H] arrays mu, sigma, d_hat, s, plus tau / alpha.
    Raises ValueError if an (layer, head) is missing or duplicated."""
    doc = path_or_doc if isinstance(path_or_doc, dict) else json.load(open(path_or_doc))
    ent = doc["entries"]
    L = 1 + max(e["layer"] for e in ent)
    H = 1 + max(e["head"] for e in ent)
    out = {k: np.full((L, H), np.nan) for k in ("mu", "sigma", "d_hat", "s")}
    seen = set()
    for e in ent:
        key = (e["layer"], e["head"])
        if key in seen:
            raise ValueError(f"duplicate schedule entry {key}")
        seen.add(key)
        out["mu"][key], out["sigma"][key] = e["mean"], e["std"]
        out["d_hat"][key], out["s"][key] = e["d_hat"], e["sparsity"]
    if len(seen) != L * H:
        raise ValueError("schedule does not cover every (layer, head) exactly once")
    out["tau"], out["alpha"] = doc["tau"], doc["alpha"]
    return out
