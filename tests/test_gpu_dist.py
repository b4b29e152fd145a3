"""GPU checks of the multi-GPU code paths that run on one device: the Ulysses resharding with a
single-rank NCCL group (pack -> all_to_all -> strided layer -> all_to_all -> unpack) must equal
the layer on the whole sequence bit for bit; head-parallel shards are checked in
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


def _fused_worker(rank, world, port, ret):
    import torch.distributed as dist
    import paper_2603_18636_b200 as pb
    from paper_2603_18636_b200.dist import PeerOutput, ulysses_layer_fused
    from synthetic import video_qkv
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        w = video_qkv(4, 16, 24, 4, 128, seed=3, device="cuda")      # N = 1536, H = 4
        budget = torch.tensor([0.2, 0.3, 0.25, 0.4], device="cuda")
        ref = pb.coclust_sparse_attention(w.q, w.k, w.v, 24, 64, 2, budget)
        N, Nl = w.q.shape[2], w.q.shape[2] // world
        blk = lambda t: t.permute(0, 2, 1, 3)[:, rank * Nl:(rank + 1) * Nl].contiguous()

        def a2a(recv, send):  # input all-to-all through host memory (gloo)
            r = torch.empty_like(send, device="cpu")
            dist.all_to_all_single(r, send.cpu())
            recv.copy_(r)

        peer = PeerOutput(Nl, 4, 128, "cuda")
        o = ulysses_layer_fused(blk(w.q), blk(w.k), blk(w.v), 24, 64, 2, budget, peer, a2a=a2a)
        torch.cuda.synchronize()
        ok = torch.equal(o, blk(ref))
        dist.barrier()
        peer.close()
        dist.destroy_process_group()
        ret.put((rank, bool(ok), ""))
    except Exception as e:  # report instead of hanging the parent
        ret.put((rank, False, repr(e)))


def test_ulysses_fused_two_processes_one_gpu():
    """World size 2 on one GPU (two processes, CUDA IPC between them, gloo for the input
    all-to-all): each rank's attention epilogue writes half of its rows into the other rank's
    token block; the device barrier over peer flags orders the reads.  Each rank's block must
    equal the single-process layer bit for bit."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    ret = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_fused_worker, args=(r, 2, port, ret)) for r in range(2)]
    for p in procs:
        p.start()
    res = []
    for _ in range(2):
        res.append(ret.get(timeout=240))
    for p in procs:
        p.join(timeout=60)
        if p.is_alive():
            p.kill()
    assert all(ok for _, ok, _ in res), res
