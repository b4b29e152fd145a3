#!/usr/bin/env python
"""Measurement sweeps of SURVEY.md §8(d) beyond the single headline line of bench.py.

  cells  : BASELINE configs[4] — Wan2.1-14B 720p, cluster counts x FIXED keep ratios; per cell the
           ms per layer, the kept-FLOP roofline fraction of the attention kernel and the clustering
           overhead share.
  layers : BASELINE configs[1] / configs[2] with the DENSITY rule (R8) and the synthetic offline
           profile: one attention layer per model layer (its own seeded Q/K/V and
           per-head budgets), mean and spread over layers.

    python scripts/sweep.py cells  [--out profiles/r01_sweep_cells.jsonl]
    python scripts/sweep.py layers --config wan1.3b_480p [--layers 30]

Timing: CUDA events on the launching stream around whole layers (inputs are larger than L2),
stage times from the library's stage events, like bench.py.  Not under a profiler.
"""
from __future__ import annotations

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
from synthetic import CONFIGS, synthetic_profile, video_qkv

RULES = {"density": 0, "as_written": 1, "fixed": 2}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    d = json.load(open(p)) if os.path.exists(p) else {}
    return d.get("bf16_tflops_sustained", 1400.0), d.get("bf16_tflops", 1590.0)


def kept_flops(q, k, kq, kk, iters, budget, tau, theta, rule, seed, ws, flags=0):
    """F_kept of one layer, from the staged entries (same kernels and bits as the fused call)."""
    st = pb.coclust_assign(q, k, kq, kk, iters, seed=seed, ws=ws, kmeans=bool(flags & pb.CLUSTER_KMEANS))
    sel = pb.block_select(st["cq"], st["ck"], st["offs_q"], st["offs_k"], budget, tau, theta, rule, ws=ws,
                          flags=flags & 3)
    n_keep, kept = sel[0], sel[1]
    B, H, N, d = q.shape
    oq = st["offs_q"].cpu().numpy().reshape(B * H, -1)
    ok = st["offs_k"].cpu().numpy().reshape(B * H, -1)
    kp = kept.cpu().numpy().reshape(B * H, kq, kk)
    nk = n_keep.cpu().numpy().reshape(-1)
    nrows = sel[2].cpu().numpy().reshape(B * H, kq) if flags & 3 else np.repeat(nk[:, None], kq, 1)
    f = 0
    for bh in range(B * H):
        sq, sk = np.diff(oq[bh]), np.diff(ok[bh])
        f += sum(int(sq[a]) * int(sk[kp[bh, a, :nrows[bh, a]]].sum()) for a in range(kq))
    return 4 * d * f, nk


def time_layer(q, k, v, kq, kk, iters, budget, tau, theta, rule, seed, ws, out, warmup, steps, flags=0):
    for _ in range(warmup):
        pb.coclust_sparse_attention(q, k, v, kq, kk, iters, budget, seed=seed, tau=tau, theta=theta, rule=rule,
                                    out=out, ws=ws, sel_flags=flags)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(steps)]
    for e in (x for row in evs for x in row):
        e.record()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    torch.cuda.synchronize()
    for i in range(steps):
        starts[i].record()
        pb.coclust_sparse_attention(q, k, v, kq, kk, iters, budget, seed=seed, tau=tau, theta=theta, rule=rule,
                                    out=out, ws=ws, stage_events=evs[i], sel_flags=flags)
    starts[steps].record()
    torch.cuda.synchronize()
    ms = starts[0].elapsed_time(starts[steps]) / steps
    avg = lambda f: sum(f(i) for i in range(steps)) / steps
    stages = {"cocluster": avg(lambda i: starts[i].elapsed_time(evs[i][0])),
              "select": avg(lambda i: evs[i][0].elapsed_time(evs[i][1])),
              "permute_v_worklist": avg(lambda i: evs[i][1].elapsed_time(evs[i][2])),
              "attention": avg(lambda i: evs[i][2].elapsed_time(evs[i][3]))}
    return ms, stages


def run_cells(a):
    dev = torch.device("cuda", 0)
    c = CONFIGS["wan14b_720p"]
    w = video_qkv(c["T"], c["Hs"], c["Ws"], c["H"], c["d"], seed=a.seed, device=dev)
    q, k, v = w.q, w.k, w.v
    B, H, N, d = q.shape
    out = torch.empty_like(q)
    ws = pb.Workspace()
    sust, burst = peaks()
    dense = 4.0 * B * H * N * N * d
    clusters = [(64, 64), (128, 128), (256, 256), (512, 512), (1024, 1024), (100, 500), (256, 1024)]
    budgets = [0.05, 0.1, 0.2, 0.3, 0.5, 0.75, 1.0]
    if a.quick:
        clusters, budgets = [(100, 500), (256, 1024)], [0.1, 0.2]
    rows = []
    fout = open(a.out, "w") if a.out else None
    for kq, kk in clusters:
        for rho in budgets:
            budget = torch.full((H,), rho, dtype=torch.float32, device=dev)
            fk, nk = kept_flops(q, k, kq, kk, a.iters, budget, a.tau, a.theta, RULES["fixed"], a.seed, ws)
            ms, stg = time_layer(q, k, v, kq, kk, a.iters, budget, a.tau, a.theta, RULES["fixed"], a.seed, ws, out,
                                 a.warmup, a.steps)
            ach = fk / (stg["attention"] * 1e-3) / 1e12
            row = {"kq": kq, "kk": kk, "rho": rho, "n_keep": int(nk[0]), "ms_layer": ms, "stages_ms": stg,
                   "kept_tflop": fk / 1e12, "kept_frac": fk / dense,
                   "attn_kept_tflops": ach, "roofline_frac_sustained": ach / sust, "roofline_frac_burst": ach / burst,
                   "layer_kept_tflops": fk / (ms * 1e-3) / 1e12, "dense_equiv_tflops": dense / (ms * 1e-3) / 1e12,
                   "clustering_share": (stg["cocluster"] + stg["select"]) / ms}
            rows.append(row)
            line = json.dumps(row)
            print(line, flush=True)
            if fout:
                fout.write(line + "\n")
                fout.flush()
    # markdown summary
    print("\n| K_q/K_k | rho | n_keep | ms/layer | attn ms | attn TF/s (kept) | frac sust. | clustering share |")
    print("|---|---|---|---|---|---|---|---|")
    for r in rows:
        print(f"| {r['kq']}/{r['kk']} | {r['rho']} | {r['n_keep']} | {r['ms_layer']:.2f} | "
              f"{r['stages_ms']['attention']:.2f} | {r['attn_kept_tflops']:.0f} | {r['roofline_frac_sustained']:.3f} | "
              f"{r['clustering_share']:.3f} |")


def run_heads(a):
    """Head-parallel scaling on one GPU: every rank's layer at P = 1, 2, 4, 8 (its H / P heads,
    global sampler keys), i.e. the per-rank work of BASELINE configs[2] without the other ranks.
    Head-parallel has no collective on the data path, so the P-GPU layer time is the max over
    ranks of these per-rank times (ranks differ only by their heads' budgets / cluster sizes).
    The (P, rank) layers are captured once (CUDA graphs over head views of one tensor) and timed
    in `--rounds` interleaved rounds; each (P, rank) reports its median over the rounds, so clock
    drift over the run (power capping) does not bias the ranks measured first or last."""
    import statistics
    dev = torch.device("cuda", 0)
    c = CONFIGS["wan14b_720p"]
    w = video_qkv(c["T"], c["Hs"], c["Ws"], c["H"], c["d"], seed=a.seed, device=dev)
    H = c["H"]
    ws = pb.Workspace()
    Ps = (1, 2, 4, 8)
    calls = {}
    for P in Ps:
        Hl = H // P
        for r in range(P) if a.all_ranks else range(1):
            sl = slice(r * Hl, (r + 1) * Hl)
            q, k, v = (t[:, sl] for t in (w.q, w.k, w.v))  # head views, no copy
            out = torch.empty(1, Hl, w.q.shape[2], c["d"], dtype=w.q.dtype, device=dev)
            budget = torch.full((Hl,), 0.2, dtype=torch.float32, device=dev)
            call = (lambda q=q, k=k, v=v, out=out, budget=budget, r=r, Hl=Hl:
                    pb.coclust_sparse_attention(q, k, v, c["kq"], c["kk"], c["iters"], budget, seed=a.seed,
                                                rule=RULES["fixed"], out=out, ws=ws, head_offset=r * Hl,
                                                heads_total=H))
            for _ in range(a.warmup):
                call()
            if a.graph:
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, capture_error_mode="thread_local"):
                    call()
                call = g.replay
                call()
            calls[(P, r)] = call
    samples = {key: [] for key in calls}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for rnd in range(a.rounds):
        keys = list(calls)
        if rnd % 2:
            keys.reverse()
        for key in keys:
            call = calls[key]
            for _ in range(2):  # re-warm after switching configurations (L2 / TLB state)
                call()
            torch.cuda.synchronize()
            e0.record()
            for _ in range(a.steps):
                call()
            e1.record()
            torch.cuda.synchronize()
            samples[key].append(e0.elapsed_time(e1) / a.steps)
    rows = []
    fout = open(a.out, "w") if a.out else None
    base = None
    for P in Ps:
        times = [statistics.median(samples[(P, r)]) for r in range(P) if (P, r) in samples]
        t = max(times)
        base = base or t
        row = {"P": P, "heads_per_rank": H // P, "ms_per_rank_max": t, "ms_per_rank": times,
               "rounds": a.rounds, "predicted_scaling_efficiency": base / (P * t)}
        rows.append(row)
        print(json.dumps(row), flush=True)
        if fout:
            fout.write(json.dumps(row) + "\n")

def run_layers(a):
    dev = torch.device("cuda", 0)
    c = CONFIGS[a.config]
    nl = a.layers
    if a.schedule:  # d_hat from the offline profiler (scripts/profile_schedule.py, NEXT-3)
        doc = json.load(open(a.schedule))
        d_hat = profiler.load_schedule(doc)["d_hat"] if "entries" in doc else doc["d_hat"]  # r01 files: dense arrays
        prof = torch.tensor(d_hat, dtype=torch.float32)[:nl]
    else:
        prof = synthetic_profile(nl, c["H"], seed=a.seed)  # [L, H]; layer 0 dense
    sust, _ = peaks()
    ws = pb.Workspace()
    rows = []
    fout = open(a.out, "w") if a.out else None
    for layer in range(nl):
        w = video_qkv(c["T"], c["Hs"], c["Ws"], c["H"], c["d"], seed=a.seed, layer=layer, device=dev)
        q, k, v = w.q, w.k, w.v
        B, H, N, d = q.shape
        out = torch.empty_like(q)
        budget = prof[layer].to(dev)
        fk, nk = kept_flops(q, k, c["kq"], c["kk"], c["iters"], budget, a.tau, a.theta, RULES["density"], a.seed, ws,
                            a.sel_flags)
        ms, stg = time_layer(q, k, v, c["kq"], c["kk"], c["iters"], budget, a.tau, a.theta, RULES["density"], a.seed,
                             ws, out, a.warmup, a.steps, a.sel_flags)
        dense = 4.0 * B * H * N * N * d
        ach = fk / (stg["attention"] * 1e-3) / 1e12
        row = {"layer": layer, "budget_mean": float(budget.mean()), "n_keep": [int(x) for x in nk],
               "ms_layer": ms, "stages_ms": stg, "kept_frac": fk / dense, "attn_kept_tflops": ach,
               "roofline_frac_sustained": ach / sust, "dense_equiv_tflops": dense / (ms * 1e-3) / 1e12}
        rows.append(row)
        line = json.dumps(row)
        print(line, flush=True)
        if fout:
            fout.write(line + "\n")
            fout.flush()
        del w, q, k, v, out
    ms = np.array([r["ms_layer"] for r in rows])
    fr = np.array([r["roofline_frac_sustained"] for r in rows])
    summ = {"config": a.config, "rule": "density", "tau": a.tau, "theta": a.theta, "sel_flags": a.sel_flags,
            "budgets": a.schedule or "synthetic_profile",
            "layers": nl,
            "ms_layer_mean": float(ms.mean()), "ms_layer_min": float(ms.min()), "ms_layer_max": float(ms.max()),
            "ms_layer_mean_excl_dense_layer0": float(ms[1:].mean()) if nl > 1 else None,
            "kept_frac_mean": float(np.mean([r["kept_frac"] for r in rows])),
            "attn_roofline_frac_sustained_mean": float(fr.mean()), "attn_roofline_frac_sustained_min": float(fr.min())}
    print(json.dumps({"summary": summ}), flush=True)
    if fout:
        fout.write(json.dumps({"summary": summ}) + "\n")


def main():
    from bench import ClockSampler
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["cells", "layers", "heads"])
    ap.add_argument("--all-ranks", action="store_true", help="heads mode: time every rank's shard")
    ap.add_argument("--graph", action="store_true", help="heads mode: time CUDA-graph replays of the layer")
    ap.add_argument("--config", default="wan1.3b_480p")
    ap.add_argument("--layers", type=int, default=30)
    ap.add_argument("--iters", type=int, default=2)
    ap.add_argument("--tau", type=float, default=0.95)
    ap.add_argument("--theta", type=float, default=0.1)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--rounds", type=int, default=5, help="heads mode: interleaved timing rounds (median)")
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--sel-flags", type=int, default=0, help="NEXT-4 selection variants (layers mode)")
    ap.add_argument("--schedule", default=None, help="layers mode: budgets = d_hat of a profiler schedule JSON")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    t0 = time.time()
    clk = ClockSampler(0)
    clk.start()
    {"cells": run_cells, "layers": run_layers, "heads": run_heads}[a.mode](a)
    c = clk.stop()
    print(json.dumps({"clocks": c}), flush=True)
    if a.out:
        with open(a.out, "a") as f:
            f.write(json.dumps({"clocks": c}) + "\n")
    print(f"# wall {time.time() - t0:.1f} s", flush=True)


if __name__ == "__main__":
    main()
