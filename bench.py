#!/usr/bin/env python
"""bench.py — SVOO co-clustered block-sparse attention layer on B200 (BASELINE.json configs[2]).

One step = one pass of the whole hot path over one attention layer (all of this rank's heads):
online co-clustering (I_max iterations) -> permutation -> block selection -> block-sparse
attention with the inverse permutation fused.  Metric = ms per attention layer (lower is better),
plus dense-equivalent TFLOP/s.  Multi-GPU: head-parallel (rank r owns heads [rH/P, (r+1)H/P)),
no collective on the data path; time = max over ranks.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config ...]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ms per attention layer + dense-equiv TFLOP/s, Wan2.1-14B 720p, 1/2/4/8 B200"
CONFIG_NAMES = {"wan14b_720p": "Wan2.1-14B 720p attention (BASELINE configs[2])",
                "wan1.3b_480p": "Wan2.1-1.3B 480p attention (BASELINE configs[1])",
                "hunyuan_720p": "HunyuanVideo 720p attention (BASELINE configs[3])",
                "toy": "toy (BASELINE configs[0])"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="wan14b_720p")
    ap.add_argument("--kq", type=int, default=100)
    ap.add_argument("--kk", type=int, default=500)
    ap.add_argument("--iters", type=int, default=2)
    ap.add_argument("--budget", type=float, default=0.2)
    ap.add_argument("--rule", choices=["fixed", "density", "as_written"], default="fixed")
    ap.add_argument("--tau", type=float, default=0.95)
    ap.add_argument("--theta", type=float, default=0.1)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--reuse-steps", type=int, default=1,
                    help="also time the clustering-reuse step (P:1261-1262) and report amortised ms")
    ap.add_argument("--sel-flags", type=int, default=0,
                    help="selection variants (NEXT-4): 1 = per-row counts (R11b), 2 = size-weighted (R9c); "
                         "256 = independent k-means partitioning (w/o On baseline, NEXT-2)")
    ap.add_argument("--parallel", choices=["head", "ulysses"], default=None,
                    help="multi-GPU split (default: ulysses for hunyuan_720p, head-parallel otherwise)")
    ap.add_argument("--ulysses-return", choices=["fused", "nccl"], default="fused",
                    help="Ulysses output path: attention epilogue stores into the owners' token blocks "
                         "(fused, CUDA IPC / NVLink) or NCCL all_to_all + unpack")
    ap.add_argument("--ulysses-overlap", choices=["on", "off"], default="off",
                    help="Ulysses in-bound: packed Q|K exchange + V's exchange on a side stream overlapping the "
                         "co-clustering (on), or one packed Q|K|V exchange (off)")
    ap.add_argument("--graph", choices=["on", "off"], default="on",
                    help="time the layer as CUDA-graph replays (one captured layer call; head-parallel)")
    return ap.parse_args()


RULES = {"density": 0, "as_written": 1, "fixed": 2}


def dist_init(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        # BENCH_BACKEND=gloo + several ranks on one GPU: a functional check of the multi-rank logic
        # on a one-GPU box (its timings mean nothing); the real runs use NCCL, one GPU per rank
        backend = os.environ.get("BENCH_BACKEND", "nccl" if args.impl == "ours" else "gloo")
        dist.init_process_group(backend)
    if os.environ.get("BENCH_BACKEND") == "gloo":
        import torch
        local = local % max(1, torch.cuda.device_count())
    return ws, rank, local


def head_range(H, world, rank):
    base, rem = divmod(H, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


# ------------------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.path = f"/tmp/bench_clocks_{os.getpid()}.csv"

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        if not rows:
            return None
        sm = sorted(float(r[1]) for r in rows if r[1].replace(".", "").isdigit())
        mx = max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        pw = sorted(float(r[3]) for r in rows if r[3].replace(".", "").isdigit())
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "power_w": pw[len(pw) // 2] if pw else None, "samples": len(rows)}


# ------------------------------------------------------------------------------ oracle baseline
# the float64 oracle timed on this host's cores on ONE COMPLETE HEAD of the workload
# (co-clustering, selection, and the attention of every one of the N query rows, grouped by query
# cluster as the oracle computes it), extrapolated x H to ms per layer (every head costs the same
# work up to its cluster sizes).  The cpu_baseline leg and the --impl reference arm time the same
# head with the same code; the reference arm spreads the head's attention over its K steps (step
# i = the query clusters a = i mod K) so each step is a bounded sample and no row is extrapolated.
class OracleHead:
    def __init__(self, w, h, kq, kk, iters, budget, rule, tau, theta, seed, H_total):
        import numpy as np
        from oracle import svoo
        f = lambda t: t.float().cpu().double().numpy()
        self.Q, self.K, self.V = f(w.q[0, h]), f(w.k[0, h]), f(w.v[0, h])
        self.args = (kq, kk, iters, budget, rule, tau, theta, seed, h, H_total)
        self.np, self.svoo = np, svoo

    def cluster(self):
        """Alg. 1 + counting sort + selection (timed)."""
        np, svoo = self.np, self.svoo
        kq, kk, iters, budget, rule, tau, theta, seed, h, H_total = self.args
        t0 = time.perf_counter()
        cc = svoo.cocluster(self.Q, self.K, kq, kk, iters, seed=seed, h=h, H=H_total)
        _, oq = svoo.counting_sort(cc.Lq, kq)
        _, ok = svoo.counting_sort(cc.Lk, kk)
        self.sel = svoo.select_blocks(cc.Cq, cc.Ck, np.diff(oq), np.diff(ok), budget, tau, theta, rule,
                                      d_head=self.Q.shape[1])
        self.Lq, self.Lk = cc.Lq, cc.Lk
        return time.perf_counter() - t0

    def attention(self, clusters):
        """The oracle's masked-softmax attention for all rows of the given query clusters (timed)."""
        np, svoo = self.np, self.svoo
        t0 = time.perf_counter()
        for a in clusters:
            rows = np.nonzero(self.Lq == a)[0]
            if rows.size:
                svoo.sparse_attention(self.Q[rows], self.K, self.V, np.full(rows.size, a), self.Lk, self.sel.kept)
        return time.perf_counter() - t0


def oracle_sample_text(H, N, kq, kk, iters, detail=""):
    return (f"one complete head of {H} (float64 oracle: Alg. 1 with {iters} iterations at {kq}/{kk} clusters, "
            f"selection, and the masked-softmax attention of all {N} query rows grouped by query cluster)"
            f"{detail}; value = per-head time x {H} heads (extrapolation over heads only)")


def bench_config(args, H, N, d, world, mode, tensor_bytes):
    """The config dict of both arms (identical for the same workload)."""
    return {"workload": CONFIG_NAMES[args.config], "B": 1, "H": H, "N": N, "d": d,
            "kq": args.kq, "kk": args.kk, "iters": args.iters, "budget": args.budget,
            "rule": args.rule, "tau": args.tau, "theta": args.theta, "sel_flags": args.sel_flags,
            "parallelism": (f"ulysses-a2a x{world} (return: {args.ulysses_return}, V overlap: {args.ulysses_overlap})" if mode == "ulysses"
                            else f"head-parallel x{world}"),
            "l2": "inputs larger than L2 (%.0f MB/tensor/rank)" % (tensor_bytes / 1e6)}


def run_reference(args):
    """--impl reference: the float64 oracle as it stands, on this host's cores (rank 0 only)."""
    from synthetic import CONFIGS, video_qkv
    world, rank, local = dist_init(args)
    if rank != 0:
        return
    c = CONFIGS[args.config]
    H, d = c["H"], c["d"]
    w = video_qkv(c["T"], c["Hs"], c["Ws"], 1, d, seed=args.seed, layer=0)  # = head 0 of the layer
    N = w.q.shape[2]
    cores = len(os.sched_getaffinity(0))
    head = OracleHead(w, 0, args.kq, args.kk, args.iters, args.budget, RULES[args.rule], args.tau, args.theta,
                      args.seed, H)
    t_cluster = head.cluster()                         # the head's clustering + selection, timed once
    for i in range(args.warmup):                       # warm-up: one (small) query cluster each
        head.attention([i % args.kq])
    K = args.steps
    t_steps = [head.attention(range(i, args.kq, K)) for i in range(K)]   # together: every row once
    head_s = t_cluster + sum(t_steps)
    ms = head_s * H * 1e3
    mode = args.parallel or ("ulysses" if (args.config == "hunyuan_720p" and world > 1) else "head")
    hl = H // world if mode == "ulysses" else (lambda r: r[1] - r[0])(head_range(H, world, 0))
    line = {"impl": "reference", "metric": METRIC, "value": ms, "unit": "ms", "n_gpus": args.gpus,
            "steps": K, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "dense_equiv_tflops": 4.0 * H * N * N * d / (ms * 1e-3) / 1e12,
            "config": bench_config(args, H, N, d, world, mode, hl * N * d * 2),
            "value_kind": "extrapolated over heads: one complete head timed, x H",
            "oracle_head_s": {"cluster_select": t_cluster, "attention": sum(t_steps)},
            "cpu_baseline": {"value": ms, "unit": "ms", "cores": cores, "kind": "oracle",
                             "sample": oracle_sample_text(H, N, args.kq, args.kk, args.iters,
                                                          f"; attention split over the {K} steps (step i = "
                                                          f"query clusters i mod {K})")},
            "e2e": {"value": ms, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------ ours
def run_ours(args):
    import numpy as np
    import torch
    import paper_2603_18636_b200 as pb
    from synthetic import CONFIGS, video_qkv

    world, rank, local = dist_init(args)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    c = CONFIGS[args.config]
    H_total, d = c["H"], c["d"]
    mode = args.parallel or ("ulysses" if (args.config == "hunyuan_720p" and world > 1) else "head")
    if mode == "ulysses":
        import torch.distributed as tdist
        if not tdist.is_initialized():  # single-process Ulysses (P = 1): a one-rank NCCL group
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29555")
            tdist.init_process_group("nccl", rank=0, world_size=1)
    # deterministic generation: every rank builds the full layer and keeps its share
    full = video_qkv(c["T"], c["Hs"], c["Ws"], H_total, d, seed=args.seed, device=dev)
    N = full.q.shape[2]
    rule = RULES[args.rule]
    ws = pb.Workspace()
    budget_all = torch.full((H_total,), args.budget, dtype=torch.float32, device=dev)
    if mode == "ulysses":
        from paper_2603_18636_b200.dist import ulysses_layer
        if H_total % world or N % world:
            raise SystemExit("Ulysses needs H and N divisible by the number of GPUs")
        Hl, Nl = H_total // world, N // world
        h0, h1 = rank * Hl, (rank + 1) * Hl
        tok = lambda t: t[0].permute(1, 0, 2)[rank * Nl:(rank + 1) * Nl].unsqueeze(0).contiguous()
        q, k, v = tok(full.q), tok(full.k), tok(full.v)          # [1, N/P, H, d] token blocks
        q_h, k_h = full.q[:, h0:h1].contiguous(), full.k[:, h0:h1].contiguous()  # for F_kept only
        kw = dict(seed=args.seed, tau=args.tau, theta=args.theta, rule=rule, ws=ws,
                  overlap_v=args.ulysses_overlap == "on")
        if args.ulysses_return == "fused":
            from paper_2603_18636_b200.dist import PeerOutput, ulysses_layer_fused
            peer = PeerOutput(Nl, H_total, d, dev)

            def step(evs=None, qq=None, kk_=None, vv=None):
                return ulysses_layer_fused(q if qq is None else qq, k if kk_ is None else kk_,
                                           v if vv is None else vv, args.kq, args.kk, args.iters, budget_all, peer,
                                           stage_events=evs, **kw)
        else:
            def step(evs=None, qq=None, kk_=None, vv=None):
                return ulysses_layer(q if qq is None else qq, k if kk_ is None else kk_, v if vv is None else vv,
                                     args.kq, args.kk, args.iters, budget_all, stage_events=evs, **kw)
    else:
        h0, h1 = head_range(H_total, world, rank)
        q, k, v = (t[:, h0:h1].contiguous() for t in (full.q, full.k, full.v))
        q_h, k_h = q, k
        out = torch.empty_like(q)
        budget = budget_all[h0:h1].contiguous()
        kw = dict(seed=args.seed, tau=args.tau, theta=args.theta, rule=rule, out=out, ws=ws, head_offset=h0,
                  heads_total=H_total, sel_flags=args.sel_flags)

        def step(evs=None, qq=None, kk_=None, vv=None):
            return pb.coclust_sparse_attention(q if qq is None else qq, k if kk_ is None else kk_,
                                               v if vv is None else vv, args.kq, args.kk, args.iters, budget,
                                               stage_events=evs, **kw)
    B = 1
    H = h1 - h0
    cpu_src = full if (world == 1 and not args.no_cpu_baseline) else None
    del full

    # kept FLOPs of this rank's heads (state recomputed through the staged entries: same kernels,
    # same bits as inside the fused call)
    st = pb.coclust_assign(q_h, k_h, args.kq, args.kk, args.iters, seed=args.seed, ws=ws, head_offset=h0,
                           heads_total=H_total, kmeans=bool(args.sel_flags & pb.CLUSTER_KMEANS))
    sel = pb.block_select(st["cq"], st["ck"], st["offs_q"], st["offs_k"], budget_all[h0:h1].contiguous(),
                          args.tau, args.theta, rule, ws=ws, flags=(args.sel_flags & 3) if mode == "head" else 0)
    n_keep, kept = sel[0], sel[1]
    torch.cuda.synchronize()
    oq = st["offs_q"].cpu().numpy().reshape(B * H, -1)
    ok = st["offs_k"].cpu().numpy().reshape(B * H, -1)
    kp = kept.cpu().numpy().reshape(B * H, args.kq, args.kk)
    nk = n_keep.cpu().numpy().reshape(-1)
    nrows = (sel[2].cpu().numpy().reshape(B * H, args.kq) if len(sel) > 2
             else np.repeat(nk[:, None], args.kq, 1))
    f_kept = 0
    for bh in range(B * H):
        sq, sk = np.diff(oq[bh]), np.diff(ok[bh])
        f_kept += int(sum(int(sq[a]) * int(sk[kp[bh, a, :nrows[bh, a]]].sum()) for a in range(args.kq)))
    f_kept *= 4 * d
    del st, sel, n_keep, kept, q_h, k_h

    for _ in range(max(args.warmup, 1)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    K = args.steps
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(K)]
    for e in (x for row in evs for x in row):
        e.record()  # torch creates the CUDA event lazily, on first record
    torch.cuda.synchronize()
    # an eager pass of K steps with the library's stage events: with --graph off it is the timed
    # region; with --graph on its total is reported as stages_ms.layer_eager
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    use_graph = args.graph == "on" and mode == "head"
    clocks = ClockSampler(local)
    if not use_graph:
        clocks.start()
        time.sleep(0.3)
    torch.cuda.synchronize()
    t_start.record()
    step_starts = []
    for i in range(K):
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record()
        step_starts.append(e0)
        step(evs[i])
    t_end.record()
    torch.cuda.synchronize()
    ms = t_start.elapsed_time(t_end) / K
    st_cluster = sum(step_starts[i].elapsed_time(evs[i][0]) for i in range(K)) / K
    st_select = sum(evs[i][0].elapsed_time(evs[i][1]) for i in range(K)) / K
    st_prep = sum(evs[i][1].elapsed_time(evs[i][2]) for i in range(K)) / K
    t_attn = sum(evs[i][2].elapsed_time(evs[i][3]) for i in range(K)) / K
    ms_eager = ms
    if use_graph:
        # the timed region: K CUDA-graph replays of the layer call (40 kernel launches become one
        # graph launch; same kernels, same buffers, same bits).  One graph per timed step, each
        # captured with its own stage events (the library records them as external event nodes
        # while capturing), so the stage and attention-kernel times below are measured inside the
        # timed region itself.
        cs = torch.cuda.Stream()
        cs.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(cs):
            step()
        torch.cuda.current_stream().wait_stream(cs)
        torch.cuda.synchronize()
        gevs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(K)]
        gstart = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
        for e in [x for row in gevs for x in row] + gstart:
            e.record()
        torch.cuda.synchronize()
        graphs = []
        for i in range(K):
            g = torch.cuda.CUDAGraph()
            # thread_local: the NCCL watchdog thread may query events while this thread captures
            with torch.cuda.graph(g, pool=graphs[0].pool() if graphs else None, capture_error_mode="thread_local"):
                step(gevs[i])
            graphs.append(g)
        for w_ in range(max(args.warmup, 1)):
            graphs[w_ % K].replay()
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        clocks.start()
        time.sleep(0.3)
        torch.cuda.synchronize()
        t_start.record()
        for i in range(K):
            gstart[i].record()
            graphs[i].replay()
        t_end.record()
        torch.cuda.synchronize()
        ms = t_start.elapsed_time(t_end) / K
        st_cluster = sum(gstart[i].elapsed_time(gevs[i][0]) for i in range(K)) / K
        st_select = sum(gevs[i][0].elapsed_time(gevs[i][1]) for i in range(K)) / K
        st_prep = sum(gevs[i][1].elapsed_time(gevs[i][2]) for i in range(K)) / K
        t_attn = sum(gevs[i][2].elapsed_time(gevs[i][3]) for i in range(K)) / K
    clk = clocks.stop()
    if world > 1:
        tt = torch.tensor([ms, t_attn], device=dev)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        ms, t_attn_max = float(tt[0]), float(tt[1])
        fk = torch.tensor([float(f_kept)], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(fk)
        f_kept_total = float(fk[0])
    else:
        f_kept_total = float(f_kept)

    # ---- e2e: host buffers in, host buffer out, through the same public call.  Consecutive calls
    # are pipelined by paper_2603_18636_b200.runtime.StreamedLayer (upload of step i+1, layer of
    # step i and download of step i-1 on three streams); every step still copies its Q, K, V from
    # pinned host memory and reads its O back inside the timed region.
    e2e = None
    if not args.no_e2e:
        from paper_2603_18636_b200.runtime import StreamedLayer
        hq, hk, hv = (t.cpu().pin_memory() for t in (q, k, v))
        hos = [torch.empty(q.shape, dtype=q.dtype).pin_memory() for _ in range(2)]
        if mode == "head":
            kwe = {k_: v_ for k_, v_ in kw.items() if k_ != "out"}

            def fn(dq, dk, dv, do):
                pb.coclust_sparse_attention(dq, dk, dv, args.kq, args.kk, args.iters, budget, out=do, **kwe)
        else:
            def fn(dq, dk, dv, do):
                do.copy_(step(qq=dq, kk_=dk, vv=dv))
        sl = StreamedLayer(fn, q.shape, dev, depth=2)
        for i in range(2):
            sl.submit(i, hq, hk, hv, hos[i % 2])
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(sl.h2d)
        for i in range(K):
            sl.submit(i, hq, hk, hv, hos[i % 2])
        b_.record(sl.d2h)
        torch.cuda.synchronize()
        e2e_ms = a.elapsed_time(b_) / K
        if world > 1:
            tt = torch.tensor([e2e_ms], device=dev)
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            e2e_ms = float(tt[0])
        nbytes = q.numel() * 2
        e2e = {"value": e2e_ms, "unit": "ms", "h2d_bytes_per_step": 3 * nbytes * world,
               "d2h_bytes_per_step": nbytes * world,
               "mode": "pipelined: upload i+1 / layer i / download i-1 on 3 streams (runtime.StreamedLayer)"}
        del hq, hk, hv, hos, sl

    # clustering reuse (NEXT-1): steps that reuse the stored clustering / selection
    reuse = None
    if args.reuse_steps and mode == "head":
        st_reuse = pb.LayerState(B, H, N, d, args.kq, args.kk, dev)
        kwc = {k_: v_ for k_, v_ in kw.items() if k_ != "out"}
        pb.coclust_sparse_attention_cached(q, k, v, args.kq, args.kk, args.iters, budget, st_reuse, True,
                                           out=out, **kwc)
        for _ in range(2):
            pb.coclust_sparse_attention_cached(q, k, v, args.kq, args.kk, args.iters, budget, st_reuse, False,
                                               out=out, **kwc)
        torch.cuda.synchronize()
        a_, b2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a_.record()
        for _ in range(K):
            pb.coclust_sparse_attention_cached(q, k, v, args.kq, args.kk, args.iters, budget, st_reuse, False,
                                               out=out, **kwc)
        b2.record()
        torch.cuda.synchronize()
        t_reuse = a_.elapsed_time(b2) / K
        if world > 1:
            tt = torch.tensor([t_reuse], device=dev)
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            t_reuse = float(tt[0])
        reuse = {"reuse_step_ms": t_reuse,
                 **{f"amortized_ms_recompute_every_{R}": (ms + (R - 1) * t_reuse) / R for R in (5, 10, 20)}}
        del st_reuse

    if rank != 0:
        return
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    peak_sust = peaks.get("bf16_tflops_sustained", 1400.0)
    peak_burst = peaks.get("bf16_tflops", 1590.0)
    f_local = float(f_kept)
    achieved = f_local / (t_attn * 1e-3) / 1e12
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "attn_traffic.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath))
            # the ncu capture is of the 40-head single-GPU launch: valid only for the same launch
            if (tj.get("config") == args.config and abs(tj.get("budget", -1) - args.budget) < 1e-9
                    and H == H_total and mode == "head" and args.kq == 100 and args.kk == 500):
                traffic = tj.get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    dense_flops = 4.0 * B * H_total * N * N * d
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        head = OracleHead(cpu_src, 0, args.kq, args.kk, args.iters, args.budget, rule, args.tau, args.theta,
                          args.seed, H_total)
        t_c = head.cluster()
        t_a = head.attention(range(args.kq))
        cpu = {"value": (t_c + t_a) * H_total * 1e3, "unit": "ms", "cores": len(os.sched_getaffinity(0)),
               "kind": "oracle", "value_kind": "extrapolated over heads: one complete head timed, x H",
               "sample": oracle_sample_text(H_total, N, args.kq, args.kk, args.iters,
                                            f" ({t_c:.1f} s clustering + selection, {t_a:.1f} s attention)")}
    line = {
        "metric": METRIC, "value": ms, "unit": "ms", "n_gpus": world, "steps": K, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic",
        "dense_equiv_tflops": dense_flops / (ms * 1e-3) / 1e12,
        "config": bench_config(args, H_total, N, d, world, mode, q.numel() * 2),
        "kept_tflop_per_layer": f_kept_total / 1e12,
        "kept_frac": f_kept_total / dense_flops,
        "stages_ms": {"cocluster": st_cluster, "select": st_select, "permute_v_worklist": st_prep,
                      "attention": t_attn, "source": ("timed region: stage events captured as external event nodes in each step's CUDA graph"
                                 if use_graph else "timed region: stage events of the eager calls"),
                      "layer_eager": ms_eager},
        "timing": "CUDA-graph replays of the layer" if use_graph else "eager calls",
        # peak: the burst cuBLAS figure (the conservative denominator: the timed region is ~0.5 s of
        # layers, shorter than the 4 s the sustained figure is measured over); the sustained one beside it
        "roofline": {"kernel": "k_bsa_fwd", "bound": "tensor", "achieved": achieved, "peak": peak_burst,
                     "unit": "TFLOP/s", "frac": achieved / peak_burst, "frac_of_sustained": achieved / peak_sust,
                     "peak_sustained": peak_sust,
                     "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst: 8192^3 cuBLAS bf16, best of 10)",
                     "traffic": traffic,
                     "algorithmic": "kept FLOPs 4*d*sum_a |Q_a| sum_{c in kept[a]} |K_c| per launch (rank 0)"},
        "layer_kept_tflops": f_kept_total / (ms * 1e-3) / 1e12,
        "gpu_launches": pb.launches_per_layer(args.iters, bool(args.sel_flags & pb.CLUSTER_KMEANS), args.kq,
                                              args.kk) * K,
        "clocks": clk, "e2e": e2e, "cpu_baseline": cpu, "clustering_reuse": reuse,
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
