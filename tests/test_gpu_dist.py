"""GPU checks of the multi-GPU code paths that run on one device: the Ulysses resharding (packed
Q|K all-to-all + V's own on a side stream -> strided layer -> all-to-all back + unpack, or the
fused peer-store return) with a single-rank NCCL group and with two processes sharing the GPU
(gloo, host-staged exchanges) must equal the layer on the whole sequence bit for bit and the
oracle's masked attention on that partition within P5; head-parallel shards are checked in
test_gpu_parity.py::test_determinism_and_head_sharding."""
import os
import socket

import pytest
import torch

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_block_transpose():
    import paper_2603_18636_b200 as pb
    x = torch.randn(6, 5, 40, device="cuda").to(torch.bfloat16)
    y = pb.block_transpose(x.view(6, -1), 6, 5)
    assert torch.equal(y.view(5, 6, 40), x.transpose(0, 1))


def test_ulysses_single_rank_equals_layer():
    import torch.distributed as dist
    import paper_2603_18636_b200 as pb
    from paper_2603_18636_b200.dist import ulysses_layer
    from synthetic import video_qkv
    if not dist.is_initialized():
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_port()}", rank=0, world_size=1)
    w = video_qkv(4, 16, 24, 4, 128, seed=2, device="cuda")          # [1, 4, 1536, 128]
    budget = torch.tensor([0.2, 0.3, 0.25, 0.4], device="cuda")
    ref = pb.coclust_sparse_attention(w.q, w.k, w.v, 24, 64, 2, budget)
    tok = lambda t: t.permute(0, 2, 1, 3).contiguous()               # [1, N, H, d] token layout
    o = ulysses_layer(tok(w.q), tok(w.k), tok(w.v), 24, 64, 2, budget)
    torch.cuda.synchronize()
    assert torch.equal(o, tok(ref))
    dist.destroy_process_group()


def test_ulysses_fused_single_rank_equals_layer():
    """Fused return path with P = 1: the epilogue stores through the peer table straight into the
    token block; must equal the layer on the whole sequence bit for bit."""
    import torch.distributed as dist
    import paper_2603_18636_b200 as pb
    from paper_2603_18636_b200.dist import PeerOutput, ulysses_layer_fused
    from synthetic import video_qkv
    if not dist.is_initialized():
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{_port()}", rank=0, world_size=1)
    w = video_qkv(4, 16, 24, 4, 128, seed=2, device="cuda")
    budget = torch.tensor([0.2, 0.3, 0.25, 0.4], device="cuda")
    ref = pb.coclust_sparse_attention(w.q, w.k, w.v, 24, 64, 2, budget)
    tok = lambda t: t.permute(0, 2, 1, 3).contiguous()
    peer = PeerOutput(w.q.shape[2], 4, 128, "cuda")
    for _ in range(2):  # two layers through the same peer block (epochs 1, 2)
        o = ulysses_layer_fused(tok(w.q), tok(w.k), tok(w.v), 24, 64, 2, budget, peer,
                                a2a=lambda recv, send: recv.copy_(send))
        torch.cuda.synchronize()
        assert torch.equal(o, tok(ref))
    peer.close()
    dist.destroy_process_group()


def test_ulysses_pack_kernel_matches_reference():
    """cs_ulysses_pack against its contract: dst[p, n, t] = src_t[n, p Hl:(p+1) Hl] (T = 1..3)."""
    import paper_2603_18636_b200 as pb
    P, Nl, H, d = 4, 37, 8, 128
    for T in (1, 2, 3):
        blocks = [torch.randn(1, Nl, H, d, device="cuda").to(torch.bfloat16) for _ in range(T)]
        got = pb.ulysses_pack(blocks, P)
        ref = torch.stack([b[0].reshape(Nl, P, H // P, d) for b in blocks], dim=2).permute(1, 0, 2, 3, 4)
        assert torch.equal(got, ref)


def test_ulysses_pack_group_kernel_matches_reference():
    """cs_ulysses_pack_group: group g of G holds heads [g Hg, (g+1) Hg) of every rank's block."""
    import paper_2603_18636_b200 as pb
    P, Nl, H, d, T = 2, 29, 8, 128, 3
    blocks = [torch.randn(1, Nl, H, d, device="cuda").to(torch.bfloat16) for _ in range(T)]
    whole = pb.ulysses_pack(blocks, P)                                   # [P, Nl, T, Hl, d]
    for G in (2, 4):
        Hg = H // P // G
        for g in range(G):
            assert torch.equal(pb.ulysses_pack(blocks, P, groups=G, group=g), whole[:, :, :, g * Hg:(g + 1) * Hg])
    with pytest.raises(ValueError):
        pb.ulysses_pack(blocks, P, groups=3)


def test_ulysses_head_groups_single_rank_equals_layer():
    """Exchange split by head groups (one all-to-all per group on a side stream, the layer of group
    g after exchange g): P = 1 over NCCL, G = 2 and 4, bit-equal to the single-call layer; and the
    fused return path with G = 2."""
    import torch.distributed as dist
    import paper_2603_18636_b200 as pb
    from paper_2603_18636_b200.dist import PeerOutput, ulysses_layer
    from synthetic import video_qkv
    if not dist.is_initialized():
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_port()}", rank=0, world_size=1)
    w = video_qkv(4, 16, 24, 4, 128, seed=6, device="cuda")
    budget = torch.tensor([0.2, 0.3, 0.25, 0.4], device="cuda")
    ref = pb.coclust_sparse_attention(w.q, w.k, w.v, 24, 64, 2, budget)
    tok = lambda t: t.permute(0, 2, 1, 3).contiguous()
    for G in (2, 4):
        o = ulysses_layer(tok(w.q), tok(w.k), tok(w.v), 24, 64, 2, budget, head_groups=G)
        torch.cuda.synchronize()
        assert torch.equal(o, tok(ref)), G
    peer = PeerOutput(w.q.shape[2], 4, 128, "cuda")
    o = ulysses_layer(tok(w.q), tok(w.k), tok(w.v), 24, 64, 2, budget, head_groups=2, peer=peer)
    torch.cuda.synchronize()
    assert torch.equal(o, tok(ref))
    peer.close()
    dist.destroy_process_group()


def _oracle_check(w, o_tok, budget, rows=256):
    """o_tok [1, N, H, d] (token layout) vs the oracle's masked attention on the single-process
    partition (the GPU's labels / kept blocks, bit-identical to the sharded run's), sampled rows."""
    import numpy as np
    import paper_2603_18636_b200 as pb
    from oracle import svoo
    st = pb.coclust_assign(w.q, w.k, 24, 64, 2)
    n_keep, kept = pb.block_select(st["cq"], st["ck"], st["offs_q"], st["offs_k"], budget, 0.95, 0.1, pb.RULE_DENSITY)
    torch.cuda.synchronize()
    f = lambda t: t.float().cpu().double().numpy()
    rng = np.random.default_rng(0)
    worst = 0.0
    for h in range(w.q.shape[1]):
        Lq, Lk = st["lq"][0, h].cpu().numpy(), st["lk"][0, h].cpu().numpy()
        n = int(n_keep[0, h])
        rs = rng.choice(w.q.shape[2], rows, replace=False)
        ref = svoo.sparse_attention(f(w.q[0, h])[rs], f(w.k[0, h]), f(w.v[0, h]), Lq[rs], Lk,
                                    kept[0, h, :, :n].cpu().numpy())
        err = np.abs(f(o_tok[0, rs, h]) - ref)
        assert err.max() <= 2e-2 and err.mean() <= 5e-3, (h, err.max(), err.mean())
        worst = max(worst, float(err.max()))
    return worst


def test_ulysses_single_rank_vs_oracle():
    """P = 1 (NCCL): both exchange layouts (packed Q|K + V overlapped, packed Q|K|V) and the oracle."""
    import torch.distributed as dist
    import paper_2603_18636_b200 as pb
    from paper_2603_18636_b200.dist import ulysses_layer
    from synthetic import video_qkv
    if not dist.is_initialized():
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_port()}", rank=0, world_size=1)
    w = video_qkv(4, 16, 24, 4, 128, seed=4, device="cuda")
    budget = torch.tensor([0.2, 0.3, 0.25, 0.4], device="cuda")
    ref = pb.coclust_sparse_attention(w.q, w.k, w.v, 24, 64, 2, budget)
    tok = lambda t: t.permute(0, 2, 1, 3).contiguous()
    for ov in (True, False):
        o = ulysses_layer(tok(w.q), tok(w.k), tok(w.v), 24, 64, 2, budget, overlap_v=ov)
        torch.cuda.synchronize()
        assert torch.equal(o, tok(ref)), ov
    _oracle_check(w, o, budget)
    dist.destroy_process_group()


def _two_rank_worker(rank, world, port, fused, ret):
    import torch.distributed as dist
    import paper_2603_18636_b200 as pb
    from paper_2603_18636_b200.dist import PeerOutput, ulysses_layer
    from synthetic import video_qkv
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        w = video_qkv(4, 16, 24, 4, 128, seed=3, device="cuda")      # N = 1536, H = 4
        budget = torch.tensor([0.2, 0.3, 0.25, 0.4], device="cuda")
        ref = pb.coclust_sparse_attention(w.q, w.k, w.v, 24, 64, 2, budget)
        N, Nl = w.q.shape[2], w.q.shape[2] // world
        blk = lambda t: t.permute(0, 2, 1, 3)[:, rank * Nl:(rank + 1) * Nl].contiguous()

        def a2a(recv, send):  # all-to-all through host memory (gloo)
            r = torch.empty_like(send, device="cpu")
            dist.all_to_all_single(r, send.cpu())
            recv.copy_(r)

        peer = PeerOutput(Nl, 4, 128, "cuda") if fused else None
        o = ulysses_layer(blk(w.q), blk(w.k), blk(w.v), 24, 64, 2, budget, a2a=a2a, peer=peer)
        torch.cuda.synchronize()
        ok = torch.equal(o, blk(ref))
        dist.barrier()
        if peer is not None:
            peer.close()
        dist.destroy_process_group()
        ret.put((rank, bool(ok), o.float().cpu().numpy() if rank == 0 else None, ""))
    except Exception as e:  # report instead of hanging the parent
        ret.put((rank, False, None, repr(e)))


@pytest.mark.parametrize("fused", [False, True])
def test_ulysses_two_processes_one_gpu(fused):
    """World size 2 on one GPU (two processes; gloo exchanges through host memory; for the fused
    return, CUDA IPC between the processes and the device barrier over peer flags).  NCCL-return
    path: pack -> packed Q|K exchange + V exchange on a side stream -> strided layer -> O exchange
    -> unpack.  Each rank's block must equal the single-process layer bit for bit, and rank 0's
    block the oracle's masked attention (P5)."""
    import torch.multiprocessing as mp
    from synthetic import video_qkv
    ctx = mp.get_context("spawn")
    ret = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_two_rank_worker, args=(r, 2, port, fused, ret)) for r in range(2)]
    for p in procs:
        p.start()
    res = [ret.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        if p.is_alive():
            p.kill()
    assert all(ok for _, ok, _, _ in res), [(r, ok, e) for r, ok, _, e in res]
    o0 = next(o for r, _, o, _ in res if r == 0)
    w = video_qkv(4, 16, 24, 4, 128, seed=3, device="cuda")
    budget = torch.tensor([0.2, 0.3, 0.25, 0.4], device="cuda")
    Nl = w.q.shape[2] // 2
    # rank 0's rows against the oracle on the single-process partition (bit-identical labels)
    import numpy as np
    import paper_2603_18636_b200 as pb
    from oracle import svoo
    st = pb.coclust_assign(w.q, w.k, 24, 64, 2)
    n_keep, kept = pb.block_select(st["cq"], st["ck"], st["offs_q"], st["offs_k"], budget, 0.95, 0.1, pb.RULE_DENSITY)
    torch.cuda.synchronize()
    f = lambda t: t.float().cpu().double().numpy()
    for h in range(4):
        Lq, Lk = st["lq"][0, h].cpu().numpy(), st["lk"][0, h].cpu().numpy()
        n = int(n_keep[0, h])
        ref = svoo.sparse_attention(f(w.q[0, h])[:Nl], f(w.k[0, h]), f(w.v[0, h]), Lq[:Nl], Lk,
                                    kept[0, h, :, :n].cpu().numpy())
        err = np.abs(o0[0, :, h].astype(np.float64) - ref)
        assert err.max() <= 2e-2 and err.mean() <= 5e-3, (h, err.max())
