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

Fused return path (`ulysses_layer_fused`): the output token blocks of all ranks are mapped into
every process (CUDA IPC; over NVLink on a multi-GPU box) and the attention epilogue stores each
output row straight into the block of the rank that owns its token — the inverse permutation,
the return all-to-all and the unpack become the attention kernel's own stores.  A device-side
barrier over peer flags (cs_peer_barrier) orders the consumer after every rank's epilogue.
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


class PeerOutput:
    """This rank's output token block [1, N/P, H, d] (bf16) and flag array, mapped into every rank
    of `group` by CUDA IPC; `ptrs` / `flag_ptrs` are int64 device tensors [P] of the mapped
    addresses (this rank's own entry is its local pointer)."""

    def __init__(self, Nl, H, d, device, group=None):
        import torch
        import torch.distributed as dist
        import paper_2603_18636_b200 as pb
        self.P = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.out = torch.zeros(1, Nl, H, d, dtype=torch.bfloat16, device=device)
        self.flags = torch.zeros(self.P, dtype=torch.int32, device=device)
        torch.cuda.synchronize(device)
        mine = (pb.ipc_handle(self.out), pb.ipc_handle(self.flags)) if self.P > 1 else None
        allh = [None] * self.P
        dist.all_gather_object(allh, mine, group=group)
        self._opened = []
        optrs, fptrs = [], []
        for p in range(self.P):
            if p == self.rank:
                optrs.append(self.out.data_ptr())
                fptrs.append(self.flags.data_ptr())
                continue
            (ho, oo), (hf, of) = allh[p]
            po, pf = pb.ipc_open(ho, oo), pb.ipc_open(hf, of)
            self._opened += [(po, oo), (pf, of)]
            optrs.append(po)
            fptrs.append(pf)
        as_i64 = lambda xs: torch.tensor([x if x < 2 ** 63 else x - 2 ** 64 for x in xs], dtype=torch.int64,
                                         device=device)
        self.ptrs, self.flag_ptrs = as_i64(optrs), as_i64(fptrs)
        self.epoch = 0

    def close(self):
        import paper_2603_18636_b200 as pb
        for p, off in self._opened:
            pb.ipc_close(p, off)
        self._opened = []


def ulysses_layer_fused(q_loc, k_loc, v_loc, kq, kk, iters, budget, peer: "PeerOutput", *, group=None,
                        a2a=None, **kw):
    """ulysses_layer with the return all-to-all fused into the attention epilogue (see module doc).

    Returns peer.out [1, N/P, H, d], complete once the calling stream passes the device barrier.
    `a2a(recv, send)` overrides the input all_to_all_single (e.g. through host memory for a gloo
    group in tests)."""
    import torch
    import torch.distributed as dist
    import paper_2603_18636_b200 as pb
    P = dist.get_world_size(group)
    r = dist.get_rank(group)
    B, Nl, H, d = q_loc.shape
    if B != 1 or H % P:
        raise ValueError("Ulysses path needs B == 1 and H divisible by the group size")
    Hl = H // P
    N = Nl * P
    a2a = a2a or (lambda recv, send: dist.all_to_all_single(recv, send, group=group))
    full = []
    for x in (q_loc, k_loc, v_loc):
        send = pb.block_transpose(x.contiguous().view(Nl, P * Hl * d), Nl, P)
        recv = torch.empty_like(send)
        a2a(recv, send)
        full.append(recv.view(N, Hl, d).permute(1, 0, 2).unsqueeze(0))
    pb.coclust_sparse_attention_peer(full[0], full[1], full[2], kq, kk, iters, budget[r * Hl:(r + 1) * Hl].contiguous(),
                                     peer_ptrs=peer.ptrs, P=P, n_per_rank=Nl, head_base=r * Hl, s_tok=H * d,
                                     s_head=d, head_offset=r * Hl, heads_total=H, **kw)
    peer.epoch += 1
    pb.peer_barrier(P, r, peer.flag_ptrs, peer.epoch, full[0])
    return peer.out
