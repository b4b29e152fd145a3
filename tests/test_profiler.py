"""NEXT-3 schedule module (paper_2603_18636_b200/profiler.py) against what the paper
and the mathematics fix: the normal quantile against scipy, the Gaussian fit against scipy's
maximum-likelihood fit, the SPEC's worked schedule examples, argument errors
(S:256-257), monotonicity in alpha, and the SPEC JSON schema round trip."""
import json

import numpy as np
import pytest
from scipy import stats

from paper_2603_18636_b200 import profiler


def test_normal_quantile_matches_scipy():
    ps = np.concatenate([[1e-12, 1e-6, 0.01, 0.02425, 0.3, 0.5, 0.9, 0.95, 0.975, 0.99, 1 - 1e-6],
                         np.random.default_rng(0).uniform(0.001, 0.999, 200)])
    for p in ps:
        assert abs(profiler.normal_quantile(float(p)) - stats.norm.ppf(p)) <= 1e-12 * max(1.0, abs(stats.norm.ppf(p)))
    assert abs(profiler.normal_quantile(0.95) - profiler.Z_ALPHA_95) < 1e-14
    for bad in (0.0, 1.0, -0.1):
        with pytest.raises(ValueError):
            profiler.normal_quantile(bad)


def test_fit_matches_scipy_mle():
    d = np.random.default_rng(1).uniform(0.01, 0.6, size=(10, 3, 4))
    s = profiler.fit_schedule(d, alpha=0.9)
    for l in range(3):
        for h in range(4):
            mu, sd = stats.norm.fit(d[:, l, h])  # maximum likelihood: ddof = 0
            assert abs(s["mu"][l, h] - mu) < 1e-14 and abs(s["sigma"][l, h] - sd) < 1e-14
            assert abs(s["d_hat"][l, h] - min(1.0, mu + stats.norm.ppf(0.9) * sd)) < 1e-12
    assert np.array_equal(s["s"], 1.0 - s["d_hat"])
    assert s["samples"].shape == (3, 4, 10) and np.array_equal(s["samples"][1, 2], d[:, 1, 2])


@pytest.mark.parametrize("samples,d_hat,sp", [([0.3, 0.3, 0.3], 0.3, 0.7),    # S:259 sigma = 0
                                              ([0.2, 0.4], 0.464485, 0.535515),
                                              ([0.9, 1.0], 1.0, 0.0)])           # S:261 clamp
def test_spec_schedule_examples(samples, d_hat, sp):
    s = profiler.fit_schedule(np.asarray(samples)[:, None, None], alpha=0.95, tau=0.95)
    assert abs(s["d_hat"][0, 0] - d_hat) <= 1e-6 and abs(s["s"][0, 0] - sp) <= 1e-6


def test_fit_argument_errors():
    with pytest.raises(ValueError):
        profiler.fit_schedule(np.zeros((0, 2, 3)))          # empty sample list
    for bad in (0.0, 1.5, np.nan):
        with pytest.raises(ValueError):
            profiler.fit_schedule(np.full((2, 1, 1), bad))
    with pytest.raises(ValueError):
        profiler.fit_schedule(np.full((2, 1, 1), 0.2), alpha=0.4)
    with pytest.raises(ValueError):
        profiler.fit_schedule(np.full((2, 1), 0.2))


def test_raising_alpha_never_lowers_d_hat():
    d = np.random.default_rng(2).uniform(0.05, 0.5, size=(6, 4, 5))
    prev = None
    for a in (0.5, 0.8, 0.9, 0.95, 0.99):
        dh = profiler.fit_schedule(d, alpha=a)["d_hat"]
        if prev is not None:
            assert np.all(dh >= prev)
        prev = dh


def test_spec_json_round_trip(tmp_path):
    d = np.random.default_rng(3).uniform(0.05, 0.5, size=(5, 3, 2))
    s = profiler.fit_schedule(d, alpha=0.95, tau=0.9)
    path = tmp_path / "schedule.json"
    profiler.save_schedule(str(path), s, meta={"config": "test"})
    doc = json.load(open(path))
    assert doc["tau"] == 0.9 and doc["alpha"] == 0.95
    keys = [(e["layer"], e["head"]) for e in doc["entries"]]
    assert keys == sorted(keys) and len(keys) == 6
    assert set(doc["entries"][0]) == {"layer", "head", "mean", "std", "d_hat", "sparsity", "samples"}
    assert doc["entries"][3]["samples"] == [float(v) for v in d[:, 1, 1]]
    back = profiler.load_schedule(str(path))
    for k in ("mu", "sigma", "d_hat", "s"):
        assert np.array_equal(back[k], s[k])
    doc["entries"].append(dict(doc["entries"][0]))
    with pytest.raises(ValueError):
        profiler.load_schedule(doc)
    doc["entries"] = doc["entries"][2:-1]
    with pytest.raises(ValueError):
        profiler.load_schedule(doc)
