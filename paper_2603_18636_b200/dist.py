"""Multi-GPU plumbing for the SVOO layer: one process per GPU, torch.distributed.

Head-parallel (BASELINE configs[2]): every step of the path is per (b, h), so rank r owns heads
[lo_r, hi_r) of the layer and runs the single-GPU layer on them with head_offset = lo_r,
heads_total = H — the R4 sampler streams are keyed by the global head, so each head's result is
bit-identical to a single-GPU run.  No collective on the data path.
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
