"""Multi-GPU plumbing for the SVOO layer: one process per GPU, torch.distributed.

Head-parallel (BASELINE configs[2]): every step of the path is per (b, h), so rank r owns heads
[lo_r, hi_r) of the layer and runs the single-GPU layer on them with head_offset = lo_r,
heads_total = H — the R4 sampler streams are keyed by the global head, so each head's result is
bit-identical to a single-GPU run.  No collective on the data path.

Ulysses (BASELINE configs[3]): each rank holds a token block [B=1, N/P, H, d] of Q, K,
V.  One all_to_all_single of the packed Q|K buffer (cs_ulysses_pack, our kernel) turns it into all
N tokens of H/P heads; the layer reads them from the receive buffer through strides (no copy).
V's all_to_all_single runs on a side stream while the layer co-clusters (Alg. 1 reads only Q and
K); the layer waits on V's event just before its V permute.  O comes back with one
all_to_all_single + unpack (cs_block_transpose) or, fused, through the attention epilogue.

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


class CudaOps:
    """The device operations of the Ulysses layer (all of them libcoclust kernels): the in-bound
    pack, the layer entry, the out-bound unpack, the device barrier, and the side stream V's
    exchange runs on.  The CPU tests substitute a reference implementation of the same contract."""

    def pack(self, blocks, P, groups=1, group=0):
        import paper_2603_18636_b200 as pb
        return pb.ulysses_pack(blocks, P, groups=groups, group=group)

    def transpose(self, x, A, B):
        import paper_2603_18636_b200 as pb
        return pb.block_transpose(x, A, B)

    def layer(self, q, k, v, kq, kk, iters, budget, **kw):
        import paper_2603_18636_b200 as pb
        return pb.coclust_sparse_attention_ulysses(q, k, v, kq, kk, iters, budget, **kw)

    def barrier(self, peer, P, r, like):
        import paper_2603_18636_b200 as pb
        pb.peer_barrier(P, r, peer.flag_ptrs, peer.epoch, like)

    def exchange_async(self, send, a2a):
        """a2a of `send` on a side stream ordered after the current stream; -> (recv, event)."""
        import torch
        cur = torch.cuda.current_stream(send.device)
        side = torch.cuda.Stream(send.device)
        side.wait_stream(cur)
        with torch.cuda.stream(side):
            recv = torch.empty_like(send)
            a2a(recv, send)
            ev = torch.cuda.Event()
            ev.record(side)
        recv.record_stream(cur)
        send.record_stream(side)
        return recv, ev

    def exchange_chain(self, sends, a2a):
        """The all-to-alls of `sends`, in order, on ONE side stream ordered after the current stream
        (one communicator, one issue order on every rank); -> [(recv, event)] per send."""
        import torch
        cur = torch.cuda.current_stream(sends[0].device)
        side = torch.cuda.Stream(sends[0].device)
        side.wait_stream(cur)
        res = []
        with torch.cuda.stream(side):
            for send in sends:
                recv = torch.empty_like(send)
                a2a(recv, send)
                ev = torch.cuda.Event()
                ev.record(side)
                recv.record_stream(cur)
                send.record_stream(side)
                res.append((recv, ev))
        return res

    def wait(self, ev):
        import torch
        torch.cuda.current_stream().wait_event(ev)


def ulysses_layer(q_loc, k_loc, v_loc, kq, kk, iters, budget, *, group=None, a2a=None, peer=None,
                  overlap_v=False, head_groups=1, ops=None, **kw):
    """Sequence-parallel SVOO layer.

    q_loc, k_loc, v_loc: [1, N/P, H, d] bf16 token blocks of this rank (rank r holds tokens
    [r N/P, (r+1) N/P)); budget: [H] float32 for the whole layer.  Returns o_loc [1, N/P, H, d].

    In-bound (default): ONE all_to_all_single of the packed Q|K|V send buffer (cs_ulysses_pack:
    per destination rank, per token, the Q, K and V head rows side by side); the layer reads its
    H/P heads straight from the receive buffer through strides.  overlap_v=True instead exchanges
    Q|K first and V in a second all_to_all_single on a side stream, overlapped with the
    co-clustering and selection (which read only Q and K): the layer's stream waits on V's event
    just before the V permute (coclust_sparse_attention_ulysses, v_ready).  On one GPU (P = 1,
    where the exchange is a local copy) that variant is erratic (occasional +10-14 ms layers) and
    not faster, so it is opt-in; its value on an NVLink box is unmeasured.
    head_groups=G > 1 splits the in-bound exchange by head groups instead: G packed
    Q|K|V buffers (cs_ulysses_pack_group, heads [g Hl/G, (g+1) Hl/G) of every rank's block), their
    all_to_alls in order on one side stream, and the layer of group g (its own call, global head
    offset r Hl + g Hl/G) waits only for exchange g — exchange g+1 overlaps layer g.  Each head's
    result is bit-identical to the single-call layer (per-head work, global sampler streams).
    Out-bound: `peer` (a PeerOutput) -> the attention epilogue stores every row straight into the
    owning rank's token block (fused return, then a device barrier); else one all_to_all_single of
    O + unpack.  `a2a(recv, send)` overrides the exchange (e.g. through host memory for a gloo
    group); `ops` overrides the device operations (CudaOps).
    """
    import torch
    import torch.distributed as dist
    ops = ops or CudaOps()
    P = dist.get_world_size(group)
    r = dist.get_rank(group)
    B, Nl, H, d = q_loc.shape
    if B != 1 or H % P:
        raise ValueError("Ulysses path needs B == 1 and H divisible by the group size")
    Hl = H // P
    N = Nl * P
    a2a = a2a or (lambda recv, send: dist.all_to_all_single(recv, send, group=group))
    blocks = [x.contiguous() for x in (q_loc, k_loc, v_loc)]
    kw.setdefault("heads_total", H)
    if head_groups > 1:
        if overlap_v or Hl % head_groups:
            raise ValueError("head_groups must divide H / P and excludes overlap_v")
        G, Hg = head_groups, Hl // head_groups
        base = kw.pop("head_offset", r * Hl)
        exch = ops.exchange_chain([ops.pack(blocks, P, groups=G, group=g) for g in range(G)], a2a)
        if peer is None:
            out_buf = torch.empty(N, Hl, d, dtype=q_loc.dtype, device=q_loc.device)
            o_view = out_buf.permute(1, 0, 2).unsqueeze(0)
        for g, (rg, ev) in enumerate(exch):
            if ev is not None:
                ops.wait(ev)
            gv = lambda t: rg.view(N, 3, Hg, d)[:, t].permute(1, 0, 2).unsqueeze(0)
            bud = budget[r * Hl + g * Hg:r * Hl + (g + 1) * Hg].contiguous()
            if peer is not None:
                ops.layer(gv(0), gv(1), gv(2), kq, kk, iters, bud, head_offset=base + g * Hg,
                          peer=dict(ptrs=peer.ptrs, P=P, n_per_rank=Nl, head_base=r * Hl + g * Hg, s_tok=H * d,
                                    s_head=d), **kw)
            else:
                ops.layer(gv(0), gv(1), gv(2), kq, kk, iters, bud, head_offset=base + g * Hg,
                          out=o_view[:, g * Hg:(g + 1) * Hg], **kw)
        if peer is not None:
            peer.epoch += 1
            ops.barrier(peer, P, r, q_loc)
            return peer.out
        back = torch.empty_like(out_buf)
        a2a(back.view(P, Nl * Hl * d), out_buf.view(P, Nl * Hl * d))
        return ops.transpose(back.view(P, Nl * Hl * d), P, Nl).view(1, Nl, H, d)
    v_ready = None
    if overlap_v:
        send_qk = ops.pack(blocks[:2], P)                        # [P, Nl, 2, Hl, d]
        recv_qk = torch.empty_like(send_qk)
        a2a(recv_qk, send_qk)                                    # first: the clustering needs it
        send_v = ops.pack(blocks[2:], P)                         # [P, Nl, 1, Hl, d]
        recv_v, v_ready = ops.exchange_async(send_v, a2a)        # overlaps the co-clustering
        T_qk, qk_buf = 2, recv_qk
        v_view = recv_v.view(N, Hl, d).permute(1, 0, 2).unsqueeze(0)   # strides (.., d, Hl d, 1)
    else:
        send = ops.pack(blocks, P)                               # [P, Nl, 3, Hl, d]
        recv = torch.empty_like(send)
        a2a(recv, send)
        T_qk, qk_buf = 3, recv
        v_view = recv.view(N, 3, Hl, d)[:, 2].permute(1, 0, 2).unsqueeze(0)
    # [N, T, Hl, d] receive buffer: tensor t is the [1, Hl, N, d] view with strides (d, T Hl d)
    view = lambda t: qk_buf.view(N, T_qk, Hl, d)[:, t].permute(1, 0, 2).unsqueeze(0)
    kw.setdefault("head_offset", r * Hl)
    bud = budget[r * Hl:(r + 1) * Hl].contiguous()
    if peer is not None:
        ops.layer(view(0), view(1), v_view, kq, kk, iters, bud, v_ready=v_ready,
                  peer=dict(ptrs=peer.ptrs, P=P, n_per_rank=Nl, head_base=r * Hl, s_tok=H * d, s_head=d), **kw)
        peer.epoch += 1
        ops.barrier(peer, P, r, q_loc)
        return peer.out
    out_buf = torch.empty(N, Hl, d, dtype=q_loc.dtype, device=q_loc.device)
    o_view = out_buf.permute(1, 0, 2).unsqueeze(0)  # written in place through strides
    ops.layer(view(0), view(1), v_view, kq, kk, iters, bud, v_ready=v_ready, out=o_view, **kw)
    back = torch.empty_like(out_buf)  # [P (source = head block), Nl, Hl, d]
    a2a(back.view(P, Nl * Hl * d), out_buf.view(P, Nl * Hl * d))
    # unpack: [P, Nl, Hl, d] -> [Nl, P, Hl, d] = [Nl, H, d]
    o_loc = ops.transpose(back.view(P, Nl * Hl * d), P, Nl)
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
    Returns peer.out [1, N/P, H, d], complete once the calling stream passes the device barrier."""
    return ulysses_layer(q_loc, k_loc, v_loc, kq, kk, iters, budget, group=group, a2a=a2a, peer=peer, **kw)
