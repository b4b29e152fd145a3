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
