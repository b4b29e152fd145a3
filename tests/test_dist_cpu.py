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


class _CpuOps:
    """Reference implementation of the Ulysses device operations (paper_2603_18636_b200.dist.CudaOps)
    with the same contracts, so the host logic (pack layout, strided views, head offsets, the two
    exchanges, unpack) runs under gloo on CPU."""

    def pack(self, blocks, P, groups=1, group=0):  # cs_ulysses_pack(_group): -> [P, Nl, T, Hg, d]
        _, Nl, H, d = blocks[0].shape
        Hg = H // P // groups
        st = torch.stack([b[0].reshape(Nl, P, H // P, d)[:, :, group * Hg:(group + 1) * Hg] for b in blocks],
                         dim=2)                                                   # [Nl, P, T, Hg, d]
        return st.permute(1, 0, 2, 3, 4).contiguous()

    def transpose(self, x, A, B):  # cs_block_transpose
        return x.reshape(A, B, -1).transpose(0, 1).contiguous().reshape(B, -1)

    def layer(self, q, k, v, kq, kk, iters, budget, out=None, peer=None, v_ready=None, head_offset=0,
              heads_total=0, **kw):
        """The layer contract (global-head sampler streams) through the oracle."""
        from oracle import svoo
        f = lambda t: t.double().numpy()
        for h in range(q.shape[1]):
            r = svoo.coclust_sparse_attention_head(f(q[0, h]), f(k[0, h]), f(v[0, h]), kq, kk, iters, 3,
                                                   float(budget[h]), 0.95, 0.1, svoo.RULE_DENSITY,
                                                   h=head_offset + h, H=heads_total)
            out[0, h].copy_(torch.from_numpy(r.O))
        return out

    def exchange_async(self, send, a2a):
        recv = torch.empty_like(send)
        a2a(recv, send)
        return recv, None

    def exchange_chain(self, sends, a2a):
        return [self.exchange_async(s_, a2a) for s_ in sends]

    def wait(self, ev):
        pass


def _ulysses_worker(rank, world, port, overlap_v, ret, head_groups=1):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2603_18636_b200.dist import ulysses_layer
    from synthetic import video_qkv
    w = video_qkv(4, 8, 8, 4, 32, seed=9)            # [1, H=4, N=256, d=32]
    N = w.q.shape[2]
    Nl = N // world
    blk = lambda t: t[0].permute(1, 0, 2)[rank * Nl:(rank + 1) * Nl].unsqueeze(0).double().contiguous()
    budget = torch.tensor([0.3, 0.2, 0.5, 0.25])
    o = ulysses_layer(blk(w.q), blk(w.k), blk(w.v), 6, 10, 2, budget, ops=_CpuOps(), overlap_v=overlap_v,
                      head_groups=head_groups)
    gathered = [None] * world
    dist.all_gather_object(gathered, (rank, o.numpy()))
    if rank == 0:
        ret.put(np.concatenate([g[1] for g in sorted(gathered, key=lambda x: x[0])], axis=1))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("overlap_v,head_groups", [(True, 1), (False, 1), (False, 2)])
def test_two_rank_ulysses_matches_single_process(overlap_v, head_groups):
    """Sequence-sharded inputs -> packed Q|K all-to-all (+ V's own, or one packed Q|K|V) -> per-head
    layer on the strided receive views -> all-to-all back + unpack == the layer run on the whole
    sequence in one process (same per-head sampler streams)."""
    from oracle import svoo
    from synthetic import video_qkv
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ulysses_worker, args=(r, world, port, overlap_v, q, head_groups))
             for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)          # [1, N, H, d]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    w = video_qkv(4, 8, 8, 4, 32, seed=9)
    budget = [0.3, 0.2, 0.5, 0.25]
    for h in range(4):
        f = lambda t: t[0, h].double().numpy()
        ref = svoo.coclust_sparse_attention_head(f(w.q), f(w.k), f(w.v), 6, 10, 2, 3, budget[h], 0.95, 0.1,
                                                 svoo.RULE_DENSITY, h=h, H=4)
        np.testing.assert_allclose(got[0, :, h, :], ref.O, atol=1e-12)


def test_ulysses_pack_layout_reference():
    """The pack contract (include/coclust.h cs_ulysses_pack) on a labelled tensor: after the
    exchange the receiver's [N, T, Hl, d] buffer holds tensor t, head p*Hl + hl of token n at
    [n, t, hl] — checked by simulating the all-to-all of P ranks' packed buffers."""
    P, Nl, Hl, d, T = 3, 4, 2, 8, 2
    H, N = P * Hl, P * Nl
    full = [torch.arange(N * H * d, dtype=torch.float64).reshape(1, N, H, d) + 1000 * t for t in range(T)]
    ops = _CpuOps()
    sends = [ops.pack([x[:, r * Nl:(r + 1) * Nl].contiguous() for x in full], P) for r in range(P)]
    for dst in range(P):
        recv = torch.cat([sends[src][dst] for src in range(P)])          # [N, T, Hl, d] (source-major)
        for t in range(T):
            assert torch.equal(recv[:, t], full[t][0, :, dst * Hl:(dst + 1) * Hl])


def test_ulysses_pack_group_layout_reference():
    """cs_ulysses_pack_group's contract: group g of G exchanges heads [g Hg, (g+1) Hg) of every
    rank's Hl-head block; the G receive buffers together hold exactly the single-pack buffer."""
    P, Nl, Hl, d, T, G = 2, 3, 4, 8, 3, 2
    H, Hg = P * Hl, Hl // G
    x = [torch.randn(1, Nl, H, d, dtype=torch.float64) for _ in range(T)]
    ops = _CpuOps()
    whole = ops.pack(x, P)                                       # [P, Nl, T, Hl, d]
    for g in range(G):
        part = ops.pack(x, P, groups=G, group=g)                 # [P, Nl, T, Hg, d]
        assert torch.equal(part, whole[:, :, :, g * Hg:(g + 1) * Hg])
