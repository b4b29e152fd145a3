"""Multi-GPU plumbing for the SVOO layer: one process per GPU, torch.distributed.

Head-parallel (BASELINE configs[2]): every step of the path is per (b, h), so rank r owns heads
[lo_r, hi_r) of the layer and runs the single-GPU layer on them with head_offset = lo_r,
heads_total = H — the R4 sampler streams are keyed by the global head, so each head's result is
bit-identical to a single-GPU run.  No collective on the data path.

Ulysses (BASELINE configs[3]): each rank holds a token block [B=1, N/P, H, d] of Q, K,
V.  One all_to_all_single per tensor (NCCL over NVLink) turns it into all N tokens of H/P heads;
the layer runs on those heads (the ABI takes the [N, H/P, d] buffer through strides, no copy);
one all_to_all_single brings O back to the token block.  The only data movement besides the
collectives is the pack / unpack block transpose (cs_block_transpose, our kernel).
"""
from __future__ import annotations


def head_range(H: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced head shard of rank `rank` (sizes differ by at most one)."""
    if not (0 <= rank < world) or H < 1:
        raise ValueError("bad shard request")
    base, rem = divmod(H, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def head_parallel_layer(q, k, v, kq, kk, iters, budget, *, rank: int, world: int, **kw):
    """Run this rank's heads of a [B, H, N, d] layer; returns (out_local [B, H_r, N, d], (lo, hi)).

    q/k/v may be the full layer (sliced here) — budget is the full [H] vector."""
    import paper_2603_18636_b200 as pb
    H = q.shape[1]
    lo, hi = head_range(H, world, rank)
    sl = slice(lo, hi)
    out = pb.coclust_sparse_attention(q[:, sl], k[:, sl], v[:, sl], kq, kk, iters,
                                      budget[sl].contiguous(), head_offset=lo, heads_total=H, **kw)
    return out, (lo, hi)


def _cuda_transpose(x, A, B):
    import paper_2603_18636_b200 as pb
    return pb.block_transpose(x, A, B)


def _cuda_layer(q, k, v, kq, kk, iters, budget, head_offset, heads_total, **kw):
    import paper_2603_18636_b200 as pb
    return pb.coclust_sparse_attention(q, k, v, kq, kk, iters, budget, head_offset=head_offset,
                                       heads_total=heads_total, **kw)


def ulysses_layer(q_loc, k_loc, v_loc, kq, kk, iters, budget, *, group=None, transpose=None,
                  layer=None, **kw):
    """Sequence-parallel SVOO layer.

    q_loc, k_loc, v_loc: [1, N/P, H, d] bf16 token blocks of this rank (rank r holds tokens
    [r N/P, (r+1) N/P)); budget: [H] float32 for the whole layer.  Returns o_loc [1, N/P, H, d].
    `transpose` / `layer` default to the CUDA library (overridable for CPU tests of the logic).
    """
    import torch
    import torch.distributed as dist
    transpose = transpose or _cuda_transpose
    layer = layer or _cuda_layer
    P = dist.get_world_size(group)
    r = dist.get_rank(group)
    B, Nl, H, d = q_loc.shape
    if B != 1 or H % P:
        raise ValueError("Ulysses path needs B == 1 and H divisible by the group size")
    Hl = H // P
    N = Nl * P
    full = []
    for x in (q_loc, k_loc, v_loc):
        # pack: [Nl, P, Hl, d] -> [P, Nl, Hl, d] (chunk p = the heads of rank p)
        send = transpose(x.contiguous().view(Nl, P * Hl * d), Nl, P)
        recv = torch.empty_like(send)  # [P (source = token block), Nl, Hl, d] == [N, Hl, d]
        dist.all_to_all_single(recv, send, group=group)
        # [N, Hl, d] buffer seen as [B=1, Hl, N, d]: strides (N Hl d, d, Hl d)
        full.append(recv.view(N, Hl, d).permute(1, 0, 2).unsqueeze(0))
    out_buf = torch.empty(N, Hl, d, dtype=q_loc.dtype, device=q_loc.device)
    o_view = out_buf.permute(1, 0, 2).unsqueeze(0)  # written in place through strides
    res = layer(full[0], full[1], full[2], kq, kk, iters, budget[r * Hl:(r + 1) * Hl].contiguous(),
                r * Hl, H, out=o_view, **kw)
    if res is not None and res.data_ptr() != o_view.data_ptr():
        o_view.copy_(res)
    back = torch.empty_like(out_buf)  # [P (source = head block), Nl, Hl, d]
    dist.all_to_all_single(back, out_buf.view(P, Nl * Hl * d), group=group)
    # unpack: [P, Nl, Hl, d] -> [Nl, P, Hl, d] = [Nl, H, d]
    o_loc = transpose(back.view(P, Nl * Hl * d), P, Nl)
    return o_loc.view(1, Nl, H, d)
