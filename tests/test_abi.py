"""C-ABI checks that need no GPU: the library loads, exports every symbol include/coclust.h
declares, and rejects bad arguments on the host before anything is launched."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2603_18636_b200 import build
    build.build()
    import paper_2603_18636_b200 as pb
    return pb.lib()


def _declared():
    src = open(os.path.join(ROOT, "include", "coclust.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(?:cs_status|int|size_t|const char\*)\s+(\w+)\s*\(", src)
    return sorted(set(names))


def test_header_declares_the_north_star_entries():
    names = _declared()
    for n in ("coclust_assign", "coclust_permute", "block_select", "block_sparse_attn",
              "coclust_sparse_attention"):
        assert n in names


def test_library_exports_every_declared_symbol(L):
    for n in _declared():
        assert hasattr(L, n), n


def test_status_strings(L):
    assert L.cs_status_string(0) == b"CS_OK"
    assert L.cs_status_string(5) == b"CS_ERR_WORKSPACE"
    assert L.cs_version() >= 100


FAKE = ctypes.c_void_p(0x10000)  # 16-byte aligned, never dereferenced (validation fails first)


def _bf16(ptr=FAKE, sb=0, sh=0, sn=128):
    import paper_2603_18636_b200 as pb
    return pb._BF16In(ptr, sb, sh, sn)


def test_permute_argument_errors(L):
    st = L.coclust_permute(1, 100, 4, None, FAKE, FAKE, FAKE, 1 << 20, None)
    assert st == 1 and b"labels" in L.cs_last_error()
    assert L.coclust_permute(0, 100, 4, FAKE, FAKE, FAKE, FAKE, 1 << 20, None) == 2
    assert L.coclust_permute(1, 100, 0, FAKE, FAKE, FAKE, FAKE, 1 << 20, None) == 3
    assert L.coclust_permute(1, 100, 1025, FAKE, FAKE, FAKE, FAKE, 1 << 20, None) == 3
    assert L.coclust_permute(1, 100, 4, FAKE, FAKE, FAKE, FAKE, 10, None) == 5
    assert L.coclust_permute(1, 100, 4, FAKE, FAKE, FAKE, None, 1 << 20, None) == 5


def test_assign_argument_errors(L):
    q = _bf16()
    args = lambda **kw: dict(dict(B=1, H=1, N=256, d=128, kq=16, kk=16, iters=2), **kw)
    def call(**kw):
        a = args(**kw)
        return L.coclust_assign(a["B"], a["H"], a["N"], a["d"], q, q, a["kq"], a["kk"], a["iters"], 0,
                                a.get("ho", 0), a.get("ht", 0), None, None, FAKE, FAKE, FAKE, FAKE, FAKE, FAKE, FAKE, FAKE,
                                FAKE, 1 << 40, None)
    assert call(d=96) == 2
    assert call(N=0) == 2
    assert call(kq=300) == 3          # kq > N
    assert call(iters=0) == 3         # I_max = 0 rejected
    assert call(kk=2000, N=4096) == 3
    assert call(ho=1) == 3            # head_offset without heads_total
    assert call(ho=3, ht=3) == 3      # offset + H > total
    bad = _bf16(ctypes.c_void_p(0x10008))
    assert L.coclust_assign(1, 1, 256, 128, bad, q, 16, 16, 2, 0, 0, 0, None, None, FAKE, FAKE, FAKE, FAKE,
                            FAKE, FAKE, FAKE, FAKE, FAKE, 1 << 40, None) == 4
    bad_stride = _bf16(sn=100)
    assert L.coclust_assign(1, 1, 256, 128, q, bad_stride, 16, 16, 2, 0, 0, 0, None, None, FAKE, FAKE, FAKE,
                            FAKE, FAKE, FAKE, FAKE, FAKE, FAKE, 1 << 40, None) == 4


def test_select_argument_errors(L):
    f = lambda tau=0.95, theta=0.1, rule=0, ws=1 << 30: L.block_select(
        1, 2, 8, 16, 64, FAKE, FAKE, FAKE, FAKE, FAKE, tau, theta, rule, FAKE, FAKE, FAKE, ws, None)
    assert f(tau=0.0) == 3 and f(tau=1.5) == 3     # tau in (0,1]
    assert f(theta=1.0) == 3
    assert f(rule=7) == 3
    assert f(ws=16) == 5


def test_attention_argument_errors(L):
    q = _bf16()
    o = __import__("paper_2603_18636_b200")._BF16Out(FAKE, 0, 0, 128)
    st = L.block_sparse_attn(1, 1, 256, 128, q, q, q, 16, 16, FAKE, FAKE, FAKE, FAKE, FAKE, FAKE,
                             0.0, o, FAKE, 1 << 40, None)
    assert st == 3  # scale must be > 0
    st = L.coclust_sparse_attention(1, 1, 256, 128, q, q, q, 16, 16, 2, 0, 0, 0, None, 0.95, 0.1, 0,
                                    0.1, o, FAKE, 1 << 40, None, None)
    assert st == 1  # budget NULL


def test_workspace_bytes_monotone(L):
    a = L.cs_workspace_bytes(1, 1, 2048, 64, 16, 16)
    b = L.cs_workspace_bytes(1, 40, 75600, 128, 100, 500)
    assert 0 < a < b
    assert L.cs_workspace_bytes(1, 1, 2048, 96, 16, 16) == 0


def test_binding_refuses_cpu_tensors():
    import torch
    import paper_2603_18636_b200 as pb
    x = torch.zeros(1, 1, 64, 64, dtype=torch.bfloat16)
    with pytest.raises(ValueError):
        pb.coclust_sparse_attention(x, x, x, 4, 4, 1, torch.ones(1))


def test_extension_entry_argument_errors(L):
    """Host-side validation of the NEXT-2/3/4 and multi-GPU entries (no launch, no GPU needed)."""
    import paper_2603_18636_b200 as pb
    q = _bf16()
    # block_select_ex: unknown flag bits; per-row counts requested without their output
    f = lambda flags, rows: L.block_select_ex(1, 2, 8, 16, 64, FAKE, FAKE, FAKE, FAKE, FAKE, 0.95, 0.1, 0, flags,
                                              FAKE, rows, FAKE, FAKE, 1 << 30, None)
    assert f(0x40, FAKE) == 3
    assert f(pb.SEL_PER_ROW, None) == 1
    # fused layer with unknown flags
    o = pb._BF16Out(FAKE, 0, 0, 128)
    st = L.coclust_sparse_attention_ex(1, 1, 256, 128, q, q, q, 16, 16, 2, 0, 0, 0, FAKE, 0.95, 0.1, 0, 0x8000,
                                       0.1, o, FAKE, 1 << 40, None, None)
    assert st == 3
    # k-means half-step: too many centroids
    assert L.kmeans_assign_step(1, 1, 256, 128, q, 2000, FAKE, FAKE, FAKE, 1 << 30, None) == 3
    # profiler: tau, passes, NULL density
    g = lambda tau=0.95, passes=0, dens=FAKE: L.attention_density(1, 1, 256, 128, q, q, tau, 0.1, passes, None,
                                                                  dens, FAKE, 1 << 30, None)
    assert g(tau=0.0) == 3 and g(passes=9) == 3 and g(dens=None) == 1
    # peer barrier bounds
    assert L.cs_peer_barrier(0, 0, FAKE, 1, None) == 3
    assert L.cs_peer_barrier(2, 2, FAKE, 1, None) == 3
    assert L.cs_peer_barrier(2, 1, FAKE, 0, None) == 3
    assert L.cs_peer_barrier(2, 1, None, 1, None) == 1
    # peer-output layer: P * n_per_rank must equal N
    po = pb._PeerOut(FAKE, 2, 100, 0, 128 * 4, 128)
    st = L.coclust_sparse_attention_peer(4, 256, 128, q, q, q, 16, 16, 2, 0, 0, 0, FAKE, 0.95, 0.1, 0, 0, 0.1,
                                         ctypes.byref(po), FAKE, 1 << 40, None, None)
    assert st == 2
    # IPC helpers refuse NULL
    assert L.cs_ipc_open(None, 0, ctypes.byref(ctypes.c_void_p())) == 1
    assert L.cs_ipc_close(None, 0) == 1
    assert L.cs_density_workspace_bytes(1, 2, 1000) > 0 and L.cs_density_workspace_bytes(0, 2, 1000) == 0


def test_broadcast_and_overlapping_strides_rejected(L):
    """a stride-0 (expand()ed) dimension of extent > 1 or overlapping rows would make
    the TMA maps and the pointer-arithmetic kernels read different rows: rejected (CS_ERR_SHAPE)
    before any launch.  Extent-1 dimensions may carry any stride."""
    ok = _bf16(sb=0, sh=256 * 128, sn=128)
    call = lambda q, B=1, H=2: L.coclust_assign(B, H, 256, 128, q, ok, 16, 16, 2, 0, 0, 0, None, None, FAKE, FAKE,
                                                FAKE, FAKE, FAKE, FAKE, FAKE, FAKE, FAKE, 1 << 40, None)
    assert call(_bf16(sb=0, sh=0, sn=128)) == 2 and b"broadcast" in L.cs_last_error()     # H = 2 over sh = 0
    assert call(_bf16(sb=0, sh=256 * 128, sn=128), B=2) == 2                               # B = 2 over sb = 0
    assert call(_bf16(sb=0, sh=256 * 128, sn=64)) == 2                                     # rows overlap
    o = __import__("paper_2603_18636_b200")._BF16Out(FAKE, 0, 0, 128)                       # H = 1: sh = 0 is fine
    q1 = _bf16(sb=0, sh=0, sn=128)
    st = L.block_sparse_attn(1, 1, 256, 128, q1, q1, q1, 16, 16, FAKE, FAKE, FAKE, FAKE, FAKE, FAKE,
                             0.1, o, None, 1 << 40, None)
    assert st == 5  # passes the stride checks, stops at the NULL workspace


def test_misaligned_workspace_rejected(L):
    q = _bf16(sb=0, sh=256 * 128, sn=128)
    st = L.coclust_assign(1, 2, 256, 128, q, q, 16, 16, 2, 0, 0, 0, None, None, FAKE, FAKE, FAKE, FAKE, FAKE,
                          FAKE, FAKE, FAKE, ctypes.c_void_p(0x10004), 1 << 40, None)
    assert st == 4 and b"workspace" in L.cs_last_error()
