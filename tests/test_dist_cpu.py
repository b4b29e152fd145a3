"""World-size-2 gloo tests of the multi-GPU host logic (no GPU): head sharding covers every head
exactly once, and per-head results computed on different ranks with global sampler keys (R4)
gather to exactly the single-process result."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_18636_b200.dist import head_range


def test_head_range_partition():
    for H in (1, 5, 24, 40):
        for world in (1, 2, 3, 4, 8):
            if world > H:
                continue
            seen = []
            for r in range(world):
                lo, hi = head_range(H, world, r)
                assert hi - lo in (H // world, H // world + 1)
                seen.extend(range(lo, hi))
            assert seen == list(range(H))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, H, ret):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import svoo
    from synthetic import video_qkv
    w = video_qkv(4, 8, 8, H, 32, seed=5)
    lo, hi = head_range(H, world, rank)
    outs = []
    for h in range(lo, hi):
        f = lambda t: t[0, h].double().numpy()
        r = svoo.coclust_sparse_attention_head(f(w.q), f(w.k), f(w.v), 6, 10, 2, 3, 0.3, 0.95, 0.1,
                                               svoo.RULE_DENSITY, h=h, H=H)
        outs.append(torch.from_numpy(r.O))
    local = torch.stack(outs).numpy()
    gathered = [None] * world
    dist.all_gather_object(gathered, (lo, local))
    if rank == 0:
        ret.put(np.concatenate([g[1] for g in sorted(gathered, key=lambda x: x[0])]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_head_parallel_matches_single_process():
    from oracle import svoo
    from synthetic import video_qkv
    H, world = 3, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, H, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    w = video_qkv(4, 8, 8, H, 32, seed=5)
    for h in range(H):
        f = lambda t: t[0, h].double().numpy()
        ref = svoo.coclust_sparse_attention_head(f(w.q), f(w.k), f(w.v), 6, 10, 2, 3, 0.3, 0.95, 0.1,
                                                 svoo.RULE_DENSITY, h=h, H=H)
        assert np.array_equal(got[h], ref.O)
