#!/usr/bin/env python
"""Offline layer-wise sparsity profiling on synthetic stacks.

For m calibration inputs (seeds) and every layer of a BASELINE config, the library's
`attention_density` (tensor-core QK^T passes, no sort) gives the per-head density at tau; the
Gaussian fit over the inputs gives d_hat = mu + z_0.95 sigma and s = 1 - d_hat, written as a
schedule JSON that `scripts/sweep.py layers --schedule` feeds to the DENSITY rule.

    python scripts/profile_schedule.py --config wan1.3b_480p --inputs 10 --out profiles/r01_schedule_wan13b.json
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import paper_2603_18636_b200 as pb
from paper_2603_18636_b200 import profiler
from synthetic import CONFIGS, video_qkv


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="wan1.3b_480p")
    ap.add_argument("--layers", type=int, default=None)
    ap.add_argument("--inputs", type=int, default=10, help="calibration inputs m (P:177: 10)")
    ap.add_argument("--tau", type=float, default=0.95)
    ap.add_argument("--passes", type=int, default=4)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    c = CONFIGS[a.config]
    L = a.layers or {"wan1.3b_480p": 30, "wan14b_720p": 40, "hunyuan_720p": 60}.get(a.config, 4)
    dev = torch.device("cuda", 0)
    ws = pb.Workspace()
    dens = np.zeros((a.inputs, L, c["H"]))
    t_prof = []
    for x in range(a.inputs):
        for layer in range(L):
            # calibration input x of layer `layer`: its own seeded Q/K (the layer structure is the
            # generator's per-layer stream, the input the seed)
            w = video_qkv(c["T"], c["Hs"], c["Ws"], c["H"], c["d"], seed=1000 + x, layer=layer, device=dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            d = pb.attention_density(w.q, w.k, tau=a.tau, passes=a.passes, ws=ws)
            e1.record()
            torch.cuda.synchronize()
            t_prof.append(e0.elapsed_time(e1))
            dens[x, layer] = d[0].cpu().numpy()
            del w
    sched = profiler.fit_schedule(dens, alpha=0.95, tau=a.tau)
    N = c["T"] * c["Hs"] * c["Ws"]
    meta = {"config": a.config, "N": N, "H": c["H"], "layers": L, "inputs": a.inputs, "tau": a.tau,
            "passes": a.passes, "z": sched["z"],
            "ms_per_layer_profile_mean": float(np.mean(t_prof)), "ms_per_layer_profile_max": float(np.max(t_prof)),
            "density_mean": float(dens.mean()), "density_min": float(dens.min()), "density_max": float(dens.max()),
            "d_hat_mean": float(sched["d_hat"].mean()),
            "input_stability_sigma_over_mu_mean": float((sched["sigma"] / sched["mu"]).mean())}
    print(json.dumps(meta), flush=True)
    if a.out:
        profiler.save_schedule(a.out, sched, meta)


if __name__ == "__main__":
    main()
