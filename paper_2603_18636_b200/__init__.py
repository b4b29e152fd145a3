"""paper_2603_18636_b200 — B200 (sm_100a) hot path of SVOO (arXiv 2603.18636).

Thin ctypes binding over libcoclust.so (include/coclust.h).  This module only marshals
arguments: torch tensors provide device memory and the current CUDA stream; every step of the
path runs in the library's CUDA kernels.  There is no CPU fallback: if the library or a CUDA
device is missing, calls raise.
"""
from __future__ import annotations

import ctypes
import os

import torch

__all__ = [
    "RULE_DENSITY", "RULE_AS_WRITTEN", "RULE_FIXED", "CoclustError", "lib", "workspace_bytes",
    "Workspace", "coclust_assign", "coclust_assign_step", "coclust_update_centroids",
    "coclust_permute", "block_select", "block_sparse_attn", "coclust_sparse_attention",
]

RULE_DENSITY, RULE_AS_WRITTEN, RULE_FIXED = 0, 1, 2
SEL_PER_ROW, SEL_SIZE_WEIGHTED = 1, 2  # block_select_ex flags (include/coclust.h, NEXT-4)
CLUSTER_KMEANS = 0x100                 # fused entries: independent k-means partitioning (NEXT-2)
_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("COCLUST_LIB", os.path.join(_HERE, "libcoclust.so"))


class CoclustError(RuntimeError):
    def __init__(self, status: int, name: str, msg: str):
        super().__init__(f"{name}: {msg}")
        self.status = status
        self.name = name


class _BF16In(ctypes.Structure):
    _fields_ = [("ptr", ctypes.c_void_p), ("sb", ctypes.c_int64), ("sh", ctypes.c_int64),
                ("sn", ctypes.c_int64)]


class _BF16Out(ctypes.Structure):
    _fields_ = [("ptr", ctypes.c_void_p), ("sb", ctypes.c_int64), ("sh", ctypes.c_int64),
                ("sn", ctypes.c_int64)]


_P = ctypes.c_void_p
_I = ctypes.c_int
_SIG = {
    "cs_version": (_I, []),
    "cs_status_string": (ctypes.c_char_p, [_I]),
    "cs_last_error": (ctypes.c_char_p, []),
    "cs_workspace_bytes": (ctypes.c_size_t, [_I, _I, _I, _I, _I, _I]),
    "coclust_assign": (_I, [_I, _I, _I, _I, _BF16In, _BF16In, _I, _I, _I, ctypes.c_uint64, _I, _I, _P, _P,
                            _P, _P, _P, _P, _P, _P, _P, _P, _P, ctypes.c_size_t, _P]),
    "coclust_assign_step": (_I, [_I, _I, _I, _I, _BF16In, _I, _P, _I, _P, _P, _P, ctypes.c_size_t, _P]),
    "kmeans_assign": (_I, [_I, _I, _I, _I, _BF16In, _BF16In, _I, _I, _I, ctypes.c_uint64, _I, _I, _P, _P,
                           _P, _P, _P, _P, _P, _P, _P, _P, _P, ctypes.c_size_t, _P]),
    "kmeans_assign_step": (_I, [_I, _I, _I, _I, _BF16In, _I, _P, _P, _P, ctypes.c_size_t, _P]),
    "coclust_update_centroids": (_I, [_I, _I, _I, _I, _BF16In, _I, _P, _P, _P, _P, _P]),
    "coclust_permute": (_I, [_I, _I, _I, _P, _P, _P, _P, ctypes.c_size_t, _P]),
    "block_select": (_I, [_I, _I, _I, _I, _I, _P, _P, _P, _P, _P, ctypes.c_double, ctypes.c_double,
                          _I, _P, _P, _P, ctypes.c_size_t, _P]),
    "block_sparse_attn": (_I, [_I, _I, _I, _I, _BF16In, _BF16In, _BF16In, _I, _I, _P, _P, _P, _P, _P,
                               _P, ctypes.c_float, _BF16Out, _P, ctypes.c_size_t, _P]),
    "coclust_sparse_attention": (_I, [_I, _I, _I, _I, _BF16In, _BF16In, _BF16In, _I, _I, _I,
                                      ctypes.c_uint64, _I, _I, _P, ctypes.c_double, ctypes.c_double, _I,
                                      ctypes.c_float, _BF16Out, _P, ctypes.c_size_t, _P, _P]),
    "block_select_ex": (_I, [_I, _I, _I, _I, _I, _P, _P, _P, _P, _P, ctypes.c_double, ctypes.c_double,
                             _I, _I, _P, _P, _P, _P, ctypes.c_size_t, _P]),
    "block_sparse_attn_ex": (_I, [_I, _I, _I, _I, _BF16In, _BF16In, _BF16In, _I, _I, _P, _P, _P, _P, _P,
                                  _P, _P, ctypes.c_float, _BF16Out, _P, ctypes.c_size_t, _P]),
    "coclust_sparse_attention_ex": (_I, [_I, _I, _I, _I, _BF16In, _BF16In, _BF16In, _I, _I, _I,
                                         ctypes.c_uint64, _I, _I, _P, ctypes.c_double, ctypes.c_double, _I,
                                         _I, ctypes.c_float, _BF16Out, _P, ctypes.c_size_t, _P, _P]),
    "cs_block_transpose": (_I, [_I, _I, ctypes.c_size_t, _P, _P, _P]),
    "cs_density_workspace_bytes": (ctypes.c_size_t, [_I, _I, _I]),
    "coclust_sparse_attention_peer": (_I, [_I, _I, _I, _BF16In, _BF16In, _BF16In, _I, _I, _I, ctypes.c_uint64, _I,
                                           _I, _P, ctypes.c_double, ctypes.c_double, _I, _I, ctypes.c_float, _P, _P,
                                           ctypes.c_size_t, _P, _P]),
    "cs_peer_barrier": (_I, [_I, _I, _P, _I, _P]),
    "coclust_sparse_attention_ulysses": (_I, [_I, _I, _I, _BF16In, _BF16In, _BF16In, _I, _I, _I, ctypes.c_uint64,
                                              _I, _I, _P, ctypes.c_double, ctypes.c_double, _I, _I, ctypes.c_float,
                                              _BF16Out, _P, _P, _P, ctypes.c_size_t, _P, _P]),
    "cs_ulysses_pack": (_I, [_I, _I, _I, _I, _I, _P, _P, _P]),
    "cs_ulysses_pack_group": (_I, [_I, _I, _I, _I, _I, _I, _I, _P, _P, _P]),
    "cs_ipc_handle": (_I, [_P, _P, ctypes.POINTER(ctypes.c_size_t)]),
    "cs_ipc_open": (_I, [_P, ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p)]),
    "cs_ipc_close": (_I, [_P, ctypes.c_size_t]),
    "attention_density": (_I, [_I, _I, _I, _I, _BF16In, _BF16In, ctypes.c_double, ctypes.c_float, _I, _P, _P, _P,
                               ctypes.c_size_t, _P]),
    "coclust_sparse_attention_cached": (_I, [_I, _I, _I, _I, _BF16In, _BF16In, _BF16In, _I, _I, _I,
                                             ctypes.c_uint64, _I, _I, _P, ctypes.c_double, ctypes.c_double,
                                             _I, _I, ctypes.c_float, _BF16Out, _P, _I, _P, ctypes.c_size_t,
                                             _P, _P]),
}

_lib = None


def lib() -> ctypes.CDLL:
    """Load libcoclust.so (raises if it was not built: `python -m paper_2603_18636_b200.build`)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built; run `python -m paper_2603_18636_b200.build`")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIG.items():
            if not hasattr(L, name):  # an older library build (A/B runs); tests check the full export list
                continue
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(status: int):
    if status != 0:
        L = lib()
        raise CoclustError(status, L.cs_status_string(status).decode(), L.cs_last_error().decode())


def _stream(t: torch.Tensor) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _bf16(t: torch.Tensor, out: bool = False):
    if t.dtype != torch.bfloat16 or t.dim() != 4 or t.stride(3) != 1:
        raise ValueError("expected a bf16 [B, H, N, d] tensor with contiguous d")
    cls = _BF16Out if out else _BF16In
    return cls(t.data_ptr(), t.stride(0), t.stride(1), t.stride(2))


def _cuda(t: torch.Tensor, name: str):
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU fallback)")


def launches_per_layer(iters: int, kmeans: bool = False, kq: int = 100, kk: int = 500) -> int:
    """Kernels the fused entry launches per layer: init_sample 1; per iteration and side: anchor
    prep 2, + 1 partial-Gamma reduction when the anchor side has > 64 centroids (k-means: 1) +
    assign GEMM 1 + counting sort 3 + centroid update 1; selection 4 (Abar, rows, count, emit);
    V permute 1; work list 1; attention 1."""
    if kmeans:
        per_iter = 2 * 6
    else:  # step A anchors on C_q (kq rows), step B on C_k (kk rows)
        per_iter = 2 * 6 + 2 + (kq > 64) + (kk > 64)
    return 1 + iters * per_iter + 4 + 1 + 1 + 1


def workspace_bytes(B, H, N, d, kq, kk) -> int:
    return int(lib().cs_workspace_bytes(B, H, N, d, kq, kk))


class Workspace:
    """Grow-only device scratch buffer (caller-owned memory for the C ABI)."""

    def __init__(self):
        self.buf = None

    def get(self, nbytes: int, device) -> torch.Tensor:
        if self.buf is None or self.buf.numel() < nbytes or self.buf.device != torch.device(device):
            self.buf = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
        return self.buf


_default_ws = Workspace()


def _ws(ws, nbytes, device):
    w = (ws or _default_ws).get(nbytes, device)
    return ctypes.c_void_p(w.data_ptr()), ctypes.c_size_t(w.numel())


def coclust_assign(q, k, kq, kk, iters, seed=0, init_q=None, init_k=None, ws=None,
                   head_offset=0, heads_total=0, kmeans=False):
    """Algorithm 1 for every (b,h) + final permutation.  Returns a dict of device tensors.
    kmeans=True: the independent k-means baseline (kmeans_assign, NEXT-2) with the same outputs."""
    _cuda(q, "q")
    B, H, N, d = q.shape
    dev = q.device
    i32 = dict(dtype=torch.int32, device=dev)
    r = dict(cq=torch.empty(B, H, kq, d, dtype=torch.float32, device=dev),
             ck=torch.empty(B, H, kk, d, dtype=torch.float32, device=dev),
             lq=torch.empty(B, H, N, **i32), lk=torch.empty(B, H, N, **i32),
             perm_q=torch.empty(B, H, N, **i32), offs_q=torch.empty(B, H, kq + 1, **i32),
             perm_k=torch.empty(B, H, N, **i32), offs_k=torch.empty(B, H, kk + 1, **i32))
    w, wn = _ws(ws, workspace_bytes(B, H, N, d, kq, kk), dev)
    _check((lib().kmeans_assign if kmeans else lib().coclust_assign)(B, H, N, d, _bf16(q), _bf16(k), kq, kk, iters, seed, head_offset,
                                heads_total, _ptr(init_q),
                                _ptr(init_k), _ptr(r["cq"]), _ptr(r["ck"]), _ptr(r["lq"]),
                                _ptr(r["lk"]), _ptr(r["perm_q"]), _ptr(r["offs_q"]),
                                _ptr(r["perm_k"]), _ptr(r["offs_k"]), w, wn, _stream(q)))
    return r


def coclust_assign_step(x, c_anchor, c_self, ws=None, labels=None):
    """One Alg. 1 assignment half-step: labels [B,H,N] int32."""
    _cuda(x, "x")
    B, H, N, d = x.shape
    ka, ks = c_anchor.shape[2], c_self.shape[2]
    labels = torch.empty(B, H, N, dtype=torch.int32, device=x.device) if labels is None else labels
    w, wn = _ws(ws, workspace_bytes(B, H, N, d, ka, ks), x.device)
    _check(lib().coclust_assign_step(B, H, N, d, _bf16(x), ka, _ptr(c_anchor.contiguous()), ks,
                                     _ptr(c_self.contiguous()), _ptr(labels), w, wn, _stream(x)))
    return labels


def kmeans_assign_step(x, c_self, ws=None, labels=None):
    """One k-means assignment (NEXT-2): labels [B,H,N] int32 = argmin_j ||x_i - c_j||."""
    _cuda(x, "x")
    B, H, N, d = x.shape
    ks = c_self.shape[2]
    labels = torch.empty(B, H, N, dtype=torch.int32, device=x.device) if labels is None else labels
    w, wn = _ws(ws, workspace_bytes(B, H, N, d, ks, ks), x.device)
    _check(lib().kmeans_assign_step(B, H, N, d, _bf16(x), ks, _ptr(c_self.contiguous()), _ptr(labels), w, wn,
                                    _stream(x)))
    return labels


def coclust_update_centroids(x, perm, offs, c_inout, x_perm=None):
    _cuda(x, "x")
    B, H, N, d = x.shape
    k = c_inout.shape[2]
    _check(lib().coclust_update_centroids(B, H, N, d, _bf16(x), k, _ptr(perm), _ptr(offs),
                                          _ptr(c_inout), _ptr(x_perm), _stream(x)))
    return c_inout


def coclust_permute(labels, k, ws=None):
    """labels [..., N] int32 -> (perm [..., N], offs [..., k+1])."""
    _cuda(labels, "labels")
    N = labels.shape[-1]
    BH = labels.numel() // N
    perm = torch.empty_like(labels)
    offs = torch.empty(*labels.shape[:-1], k + 1, dtype=torch.int32, device=labels.device)
    w, wn = _ws(ws, BH * ((N + 1023) // 1024 + 1) * k * 4 + 4096, labels.device)
    _check(lib().coclust_permute(BH, N, k, _ptr(labels), _ptr(perm), _ptr(offs), w, wn,
                                 _stream(labels)))
    return perm, offs


def block_select(cq, ck, offs_q, offs_k, budget, tau=0.95, theta=0.1, rule=RULE_DENSITY, ws=None,
                 flags=0):
    """-> (n_keep [B,H] int32, kept [B,H,kq,kk] int32; first n_keep entries per row valid).
    flags (SEL_PER_ROW | SEL_SIZE_WEIGHTED, NEXT-4) != 0 -> block_select_ex, and the result gets a
    third element n_keep_rows [B,H,kq] (row a of kept holds n_keep_rows[a] entries)."""
    _cuda(cq, "cq")
    B, H, kq, d = cq.shape
    kk = ck.shape[2]
    n_keep = torch.empty(B, H, dtype=torch.int32, device=cq.device)
    kept = torch.full((B, H, kq, kk), -1, dtype=torch.int32, device=cq.device)
    w, wn = _ws(ws, B * H * kq * (kk + 1) * 4 + B * H * kq * kk * 8 + 4096, cq.device)
    if flags:
        n_rows = torch.empty(B, H, kq, dtype=torch.int32, device=cq.device)
        _check(lib().block_select_ex(B, H, kq, kk, d, _ptr(cq.contiguous()), _ptr(ck.contiguous()),
                                     _ptr(offs_q), _ptr(offs_k), _ptr(budget), float(tau), float(theta),
                                     int(rule), int(flags), _ptr(n_keep), _ptr(n_rows), _ptr(kept), w, wn,
                                     _stream(cq)))
        return n_keep, kept, n_rows
    _check(lib().block_select(B, H, kq, kk, d, _ptr(cq.contiguous()), _ptr(ck.contiguous()),
                              _ptr(offs_q), _ptr(offs_k), _ptr(budget), float(tau), float(theta),
                              int(rule), _ptr(n_keep), _ptr(kept), w, wn, _stream(cq)))
    return n_keep, kept


def block_sparse_attn(q, k, v, perm_q, offs_q, perm_k, offs_k, n_keep, kept, scale=None,
                      out=None, ws=None, n_keep_rows=None):
    """n_keep_rows [B,H,kq] (per-row counts from block_select(flags=SEL_PER_ROW)) -> the _ex entry."""
    _cuda(q, "q")
    B, H, N, d = q.shape
    kq, kk = offs_q.shape[-1] - 1, offs_k.shape[-1] - 1
    scale = d ** -0.5 if scale is None else scale
    out = torch.empty(B, H, N, d, dtype=torch.bfloat16, device=q.device) if out is None else out
    w, wn = _ws(ws, workspace_bytes(B, H, N, d, kq, kk), q.device)
    if n_keep_rows is not None:
        _check(lib().block_sparse_attn_ex(B, H, N, d, _bf16(q), _bf16(k), _bf16(v), kq, kk, _ptr(perm_q),
                                          _ptr(offs_q), _ptr(perm_k), _ptr(offs_k), _ptr(n_keep),
                                          _ptr(n_keep_rows), _ptr(kept), float(scale), _bf16(out, True), w, wn,
                                          _stream(q)))
        return out
    _check(lib().block_sparse_attn(B, H, N, d, _bf16(q), _bf16(k), _bf16(v), kq, kk, _ptr(perm_q),
                                   _ptr(offs_q), _ptr(perm_k), _ptr(offs_k), _ptr(n_keep),
                                   _ptr(kept), float(scale), _bf16(out, True), w, wn, _stream(q)))
    return out


def coclust_sparse_attention(q, k, v, kq, kk, iters, budget, *, seed=0, tau=0.95, theta=0.1,
                             rule=RULE_DENSITY, scale=None, out=None, ws=None, head_offset=0,
                             heads_total=0, stage_events=None, sel_flags=0):
    """The whole SVOO attention layer (north_star stages 1-5) on device.

    stage_events: optional 4 torch.cuda.Event (enable_timing) recorded after co-clustering,
    after selection, and around the attention kernel.  sel_flags: SEL_* selection variants
    (NEXT-4) -> coclust_sparse_attention_ex."""
    _cuda(q, "q")
    B, H, N, d = q.shape
    scale = d ** -0.5 if scale is None else scale
    out = torch.empty(B, H, N, d, dtype=torch.bfloat16, device=q.device) if out is None else out
    w, wn = _ws(ws, workspace_bytes(B, H, N, d, kq, kk), q.device)
    evs = None
    if stage_events is not None:
        evs = (ctypes.c_void_p * 4)(*[ctypes.c_void_p(e.cuda_event) for e in stage_events])
    if sel_flags:
        _check(lib().coclust_sparse_attention_ex(B, H, N, d, _bf16(q), _bf16(k), _bf16(v), kq, kk, iters,
                                                 seed, head_offset, heads_total, _ptr(budget), float(tau),
                                                 float(theta), int(rule), int(sel_flags), float(scale),
                                                 _bf16(out, True), w, wn, _stream(q), evs))
        return out
    _check(lib().coclust_sparse_attention(B, H, N, d, _bf16(q), _bf16(k), _bf16(v), kq, kk, iters,
                                          seed, head_offset, heads_total, _ptr(budget), float(tau), float(theta), int(rule),
                                          float(scale), _bf16(out, True), w, wn, _stream(q), evs))
    return out


def attention_density(q, k, tau=0.95, scale=None, passes=0, counts=False, ws=None):
    """Offline profiling (NEXT-3): attention density per (b,h) of softmax(q k^T scale)
    at mass tau -> float64 [B,H] (and the per-row prefix sizes int32 [B,H,N] if counts)."""
    _cuda(q, "q")
    B, H, N, d = q.shape
    scale = d ** -0.5 if scale is None else scale
    dens = torch.empty(B, H, dtype=torch.float64, device=q.device)
    cnt = torch.empty(B, H, N, dtype=torch.int32, device=q.device) if counts else None
    w, wn = _ws(ws, int(lib().cs_density_workspace_bytes(B, H, N)), q.device)
    _check(lib().attention_density(B, H, N, d, _bf16(q), _bf16(k), float(tau), float(scale), int(passes),
                                   _ptr(cnt), _ptr(dens), w, wn, _stream(q)))
    return (dens, cnt) if counts else dens


class _PeerOut(ctypes.Structure):
    _fields_ = [("ptrs", ctypes.c_void_p), ("P", ctypes.c_int), ("n_per_rank", ctypes.c_int),
                ("head_base", ctypes.c_int), ("s_tok", ctypes.c_int64), ("s_head", ctypes.c_int64)]


def coclust_sparse_attention_peer(q, k, v, kq, kk, iters, budget, *, peer_ptrs, P, n_per_rank, head_base,
                                  s_tok, s_head, seed=0, tau=0.95, theta=0.1, rule=RULE_DENSITY, flags=0,
                                  scale=None, ws=None, head_offset=0, heads_total=0, stage_events=None):
    """The layer (B = 1) with every output row stored straight into the token block of the rank
    that owns the token (fused Ulysses return all-to-all).  peer_ptrs: int64 device tensor [P]."""
    _cuda(q, "q")
    B, H, N, d = q.shape
    if B != 1:
        raise ValueError("peer-output layer needs B == 1")
    scale = d ** -0.5 if scale is None else scale
    w, wn = _ws(ws, workspace_bytes(B, H, N, d, kq, kk), q.device)
    po = _PeerOut(peer_ptrs.data_ptr(), P, n_per_rank, head_base, s_tok, s_head)
    evs = None
    if stage_events is not None:
        evs = (ctypes.c_void_p * 4)(*[ctypes.c_void_p(e.cuda_event) for e in stage_events])
    _check(lib().coclust_sparse_attention_peer(H, N, d, _bf16(q), _bf16(k), _bf16(v), kq, kk, iters, seed,
                                               head_offset, heads_total, _ptr(budget), float(tau), float(theta),
                                               int(rule), int(flags), float(scale), ctypes.byref(po), w, wn,
                                               _stream(q), evs))


def coclust_sparse_attention_ulysses(q, k, v, kq, kk, iters, budget, *, out=None, peer=None, v_ready=None,
                                     seed=0, tau=0.95, theta=0.1, rule=RULE_DENSITY, flags=0, scale=None, ws=None,
                                     head_offset=0, heads_total=0, stage_events=None):
    """The Ulysses layer entry (B = 1): q/k/v are [1, H, N, d] strided views of the in-bound
    all-to-all buffers.  v_ready: torch.cuda.Event the layer's stream waits on before V is first
    read (V's all-to-all overlaps the co-clustering); peer: dict(ptrs, P, n_per_rank, head_base,
    s_tok, s_head) for the fused return path (else the output goes to `out`)."""
    _cuda(q, "q")
    B, H, N, d = q.shape
    if B != 1:
        raise ValueError("the Ulysses layer entry needs B == 1")
    scale = d ** -0.5 if scale is None else scale
    po = None
    if peer is not None:
        po = _PeerOut(peer["ptrs"].data_ptr(), peer["P"], peer["n_per_rank"], peer["head_base"], peer["s_tok"],
                      peer["s_head"])
        o = _BF16Out(None, 0, 0, 0)
    else:
        out = torch.empty(B, H, N, d, dtype=torch.bfloat16, device=q.device) if out is None else out
        o = _bf16(out, True)
    w, wn = _ws(ws, workspace_bytes(B, H, N, d, kq, kk), q.device)
    evs = None
    if stage_events is not None:
        evs = (ctypes.c_void_p * 4)(*[ctypes.c_void_p(e.cuda_event) for e in stage_events])
    _check(lib().coclust_sparse_attention_ulysses(H, N, d, _bf16(q), _bf16(k), _bf16(v), kq, kk, iters, seed,
                                                  head_offset, heads_total, _ptr(budget), float(tau), float(theta),
                                                  int(rule), int(flags), float(scale), o,
                                                  ctypes.byref(po) if po is not None else None,
                                                  ctypes.c_void_p(v_ready.cuda_event) if v_ready is not None else None,
                                                  w, wn, _stream(q), evs))
    return out


def ulysses_pack(blocks, P, out=None, groups=1, group=0):
    """T rank-local token blocks [1, Nl, P*Hl, d] (bf16, contiguous) -> [P, Nl, T, Hg, d] (one send
    buffer for a single all_to_all_single of all T tensors); Hg = Hl / groups: only the heads
    [group Hg, (group+1) Hg) of every rank's Hl-head block (groups = 1: all of them)."""
    x0 = blocks[0]
    _cuda(x0, "blocks[0]")
    _, Nl, H, d = x0.shape
    T = len(blocks)
    if H % P:
        raise ValueError("H must be divisible by P")
    Hl = H // P
    if groups < 1 or Hl % groups or not 0 <= group < groups:
        raise ValueError("groups must divide H / P and 0 <= group < groups")
    Hg = Hl // groups
    for b in blocks:
        if b.shape != x0.shape or not b.is_contiguous() or b.dtype != torch.bfloat16:
            raise ValueError("blocks must be contiguous bf16 tensors of one shape")
    out = torch.empty(P, Nl, T, Hg, d, dtype=torch.bfloat16, device=x0.device) if out is None else out
    srcs = (ctypes.c_void_p * T)(*[b.data_ptr() for b in blocks])
    _check(lib().cs_ulysses_pack_group(Nl, P, Hl, Hg, group, d, T, srcs, _ptr(out), _stream(x0)))
    return out


def peer_barrier(P, rank, flag_ptrs, epoch, stream_of):
    """Device-side barrier over the peers' flag arrays (flag_ptrs: int64 device tensor [P])."""
    _check(lib().cs_peer_barrier(P, rank, _ptr(flag_ptrs), int(epoch), _stream(stream_of)))


def ipc_handle(t):
    """-> (64-byte cudaIpcMemHandle of t's allocation, byte offset of t in it)."""
    h = ctypes.create_string_buffer(64)
    off = ctypes.c_size_t(0)
    _check(lib().cs_ipc_handle(_ptr(t), h, ctypes.byref(off)))
    return h.raw, int(off.value)


def ipc_open(handle: bytes, offset: int) -> int:
    p = ctypes.c_void_p(0)
    _check(lib().cs_ipc_open(ctypes.create_string_buffer(handle, 64), offset, ctypes.byref(p)))
    return int(p.value)


def ipc_close(ptr: int, offset: int):
    _check(lib().cs_ipc_close(ctypes.c_void_p(ptr), offset))


def block_transpose(src, A, B, out=None):
    """dst[b][a] = src[a][b] over an [A, B] grid of equal rows (Ulysses pack / unpack)."""
    _cuda(src, "src")
    row_bytes = src.numel() * src.element_size() // (A * B)
    out = torch.empty(B, src.numel() // B, dtype=src.dtype, device=src.device) if out is None else out
    _check(lib().cs_block_transpose(A, B, row_bytes, _ptr(src), _ptr(out), _stream(src)))
    return out


class _LayerState(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("cq", "ck", "lq", "lk", "perm_q", "perm_k", "offs_q",
                                               "offs_k", "n_keep", "kept", "n_keep_rows")]


class LayerState:
    """Device buffers of the clustering-reuse state (cs_layer_state) for one layer."""

    def __init__(self, B, H, N, d, kq, kk, device):
        i32 = dict(dtype=torch.int32, device=device)
        self.cq = torch.empty(B, H, kq, d, dtype=torch.float32, device=device)
        self.ck = torch.empty(B, H, kk, d, dtype=torch.float32, device=device)
        self.lq, self.lk = torch.empty(B, H, N, **i32), torch.empty(B, H, N, **i32)
        self.perm_q, self.perm_k = torch.empty(B, H, N, **i32), torch.empty(B, H, N, **i32)
        self.offs_q = torch.empty(B, H, kq + 1, **i32)
        self.offs_k = torch.empty(B, H, kk + 1, **i32)
        self.n_keep = torch.empty(B, H, **i32)
        self.kept = torch.empty(B, H, kq, kk, **i32)
        self.n_keep_rows = torch.empty(B, H, kq, **i32)
        self._c = _LayerState(*[t.data_ptr() for t in (self.cq, self.ck, self.lq, self.lk, self.perm_q,
                                                        self.perm_k, self.offs_q, self.offs_k, self.n_keep,
                                                        self.kept, self.n_keep_rows)])


def coclust_sparse_attention_cached(q, k, v, kq, kk, iters, budget, state, recompute, *, seed=0, tau=0.95,
                                    theta=0.1, rule=RULE_DENSITY, scale=None, out=None, ws=None,
                                    head_offset=0, heads_total=0, stage_events=None, sel_flags=0):
    """The layer with clustering reuse: recompute=True refreshes `state`."""
    _cuda(q, "q")
    B, H, N, d = q.shape
    scale = d ** -0.5 if scale is None else scale
    out = torch.empty(B, H, N, d, dtype=torch.bfloat16, device=q.device) if out is None else out
    w, wn = _ws(ws, workspace_bytes(B, H, N, d, kq, kk), q.device)
    evs = None
    if stage_events is not None:
        evs = (ctypes.c_void_p * 4)(*[ctypes.c_void_p(e.cuda_event) for e in stage_events])
    _check(lib().coclust_sparse_attention_cached(B, H, N, d, _bf16(q), _bf16(k), _bf16(v), kq, kk, iters,
                                                 seed, head_offset, heads_total, _ptr(budget), float(tau),
                                                 float(theta), int(rule), int(sel_flags), float(scale),
                                                 _bf16(out, True), ctypes.byref(state._c), int(bool(recompute)), w, wn,
                                                 _stream(q), evs))
    return out
