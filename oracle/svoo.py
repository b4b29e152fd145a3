"""ORACLE for the SVOO hot path (arXiv 2603.18636) — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline / --impl reference
legs may import this module.  The product path (`paper_2603_18636_b200`) never imports it and
shares no code, header, table or constant generator with it.

Plain, slow, obviously-correct float64 numpy.  Every function follows the paper in its order
and notation; citations are PAPER.md line numbers ("P:n", Section / Algorithm / Eq.) and, for
the readings the paper leaves open, the DESIGN.md reading ids R1..R17 (which restate
SURVEY.md §8c).  Inputs are the exact bf16 values the GPU path also consumes, widened to fp64.

Functions and their pins (tests/test_oracle_*.py):
  splitmix64_next / sample_anchor_indices   R4            pinned: published splitmix64 vectors
                                                          (seeds 0 and 1234567), literal stream
                                                          seeds and Floyd draws derived by hand,
                                                          distinctness/range/uniformity
  l2_normalize_rows, softmax_row                           pinned: SPEC worked examples (golden)
  assign_step (Alg.1 Step A/B assignment)   P:1214-1226   pinned: cosine nearest-centroid special
                                                          case, brute-force 2-partition, K=1,
                                                          explicit-difference distances, closed-
                                                          form gap (unsquared distances)
  update_centroids (Alg.1 Mean)             P:1219,1227   pinned: member-mean / sum invariants
  cocluster (Alg.1)                         P:1203-1229   pinned: hand-derived 2-D examples
                                                          (tests/golden/alg1_examples.json): the
                                                          Fig. 3 coupling construction,
                                                          two full iterations with the centroid
                                                          generation of every half-step and the
                                                          returned (post-update, R13) centroids;
                                                          token-order invariance; R13 member means
  counting_sort                             implied P:1266 pinned: np.argsort(kind="stable")
  select_blocks (Ā, Recall, ρ rule, top-ρK)  P:1247-1257   pinned: SPEC worked examples, nesting,
                                                          hand examples of n_rec (ceil over K_q')
                                                          and of both DENSITY branches;
    + NEXT-4 variants (per_row, size_weighted)            pinned: reduce to the base reading
                                                          (FIXED / equal sizes), closed-form
                                                          size-weighted masses, hand example
  sparse_attention                          P:1257        pinned: ρ=1 == library SDPA, singleton
                                                          case, n=8 brute force, convexity
  kmeans / cocluster_kmeans ("w/o On")      P:1058, P:1270 pinned: sklearn KMeans (lloyd, same init),
                                                          Lloyd objective non-increasing
  reference_pairs / block_pair_* (recall)   P:181-183     pinned: brute-force minimal prefix,
                                                          identity / single-block partitions
  attention_density / sparsity_schedule     P:1176-1191   pinned: uniform / one-hot / geometric
                                                          rows (closed forms), brute-force minimal
                                                          subsets, scipy norm.ppf(0.95)
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

MASK64 = (1 << 64) - 1
GOLDEN_GAMMA = 0x9E3779B97F4A7C15

RULE_DENSITY = 0
RULE_AS_WRITTEN = 1
RULE_FIXED = 2


# ----------------------------------------------------------------------------------------------
# R4 — Sample(Q, K_q) (Alg. 1 line 1; "randomly sampling anchor tokens")
# ----------------------------------------------------------------------------------------------
def splitmix64_next(state: int) -> tuple[int, int]:
    """One splitmix64 step (Steele, Lea & Flood 2014).  Returns (new_state, output)."""
    state = (state + GOLDEN_GAMMA) & MASK64
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return state, z ^ (z >> 31)


def sample_seed(seed: int, b: int, h: int, H: int, side: int) -> int:
    """R4 stream seed: seed ^ (((b*H+h)*2+side) * 0x9E3779B97F4A7C15) mod 2^64."""
    return (seed ^ ((((b * H + h) * 2 + side) * GOLDEN_GAMMA) & MASK64)) & MASK64


def sample_anchor_indices(N: int, K: int, seed: int, b: int, h: int, H: int, side: int) -> np.ndarray:
    """Uniform K-subset of {0..N-1} without replacement by Floyd's algorithm (R4).

    for j = N-K .. N-1:  t = next() % (j+1);  insert (j if t already chosen else t).
    Returned ascending; centroid j is token idx[j].  side 0 = queries, 1 = keys.
    """
    if not (1 <= K <= N):
        raise ValueError("need 1 <= K <= N")
    state = sample_seed(seed, b, h, H, side)
    chosen: set[int] = set()
    for j in range(N - K, N):
        state, r = splitmix64_next(state)
        t = r % (j + 1)
        chosen.add(j if t in chosen else t)
    return np.array(sorted(chosen), dtype=np.int64)


# ----------------------------------------------------------------------------------------------
# Norm(.) (R1) and softmax (P:1118 / R7)
# ----------------------------------------------------------------------------------------------
def l2_normalize_rows(M: np.ndarray) -> np.ndarray:
    """Row-wise L2 normalisation; an all-zero row passes through unchanged (R1)."""
    M = np.asarray(M, dtype=np.float64)
    nrm = np.sqrt((M * M).sum(axis=1))
    out = M.copy()
    nz = nrm > 0
    out[nz] = M[nz] / nrm[nz, None]
    return out


def softmax_row(z: np.ndarray) -> np.ndarray:
    """softmax with max subtraction; -inf entries get probability 0."""
    z = np.asarray(z, dtype=np.float64)
    m = np.max(z)
    e = np.exp(z - m)
    return e / e.sum()


# ----------------------------------------------------------------------------------------------
# Algorithm 1, one assignment half-step (Step A: P:1214-1218; Step B: P:1222-1226)
# ----------------------------------------------------------------------------------------------
@dataclass
class AssignResult:
    labels: np.ndarray      # int64 [N]
    gap: np.ndarray         # (D_(2) - D_(1)) / D_(2)   (unsquared distances)
    dist_best: np.ndarray   # D_(1)
    objective: float        # J = sum_i D_{i, L(i)}


def assign_step(X: np.ndarray, C_anchor: np.ndarray, C_self: np.ndarray) -> AssignResult:
    """Alg. 1 assignment with anchors C_anchor (the other side) and self centroids C_self.

    Step A (keys):    P_k = K C_q^T ; Pbar_k = C_k C_q^T ; Norm both ; L_k = argmin_j ||P_k - Pbar_k[j]||_2
    Step B (queries): P_q = Q C_k^T ; Pbar_q = C_q C_k^T ; Norm both ; L_q = argmin_j ||P_q - Pbar_q[j]||_2
    Norm = row L2 (R1), normalisation applied to the final affinity rows (R3), ties -> lowest j (R2).
    The Euclidean distance is evaluated as sqrt(|a|^2 + |b|^2 - 2 a.b) with a matmul for the
    cross term (a library primitive used as a step); tests check it against explicit differences.
    |a|^2 of a Norm'ed row is exactly 1 (0 for a zero row, R1) and is used as such, so a zero
    affinity row is at distance exactly 1 from every nonzero row and its tie goes to the lowest j
    (R2) instead of being decided by the last ulp of a rounded |b|^2.
    """
    X = np.asarray(X, np.float64)
    Ca = np.asarray(C_anchor, np.float64)
    Cs = np.asarray(C_self, np.float64)
    P = X @ Ca.T                      # affinity of each token to the anchors       [N, K_a]
    Pbar = Cs @ Ca.T                  # affinity of each self centroid to anchors   [K_s, K_a]
    Ph = l2_normalize_rows(P)
    Pbh = l2_normalize_rows(Pbar)
    na = np.any(P != 0, axis=1).astype(np.float64)      # |P^_i|^2 in {0, 1}
    nb = np.any(Pbar != 0, axis=1).astype(np.float64)   # |Pbar^_j|^2 in {0, 1}
    sq = na[:, None] + nb[None, :] - 2.0 * (Ph @ Pbh.T)
    D = np.sqrt(np.maximum(sq, 0.0))  # [N, K_s]
    labels = np.argmin(D, axis=1)     # first minimum -> lowest index on ties
    N, Ks = D.shape
    d1 = D[np.arange(N), labels]
    if Ks > 1:
        D2 = D.copy()
        D2[np.arange(N), labels] = np.inf
        d2 = D2.min(axis=1)
        gap = (d2 - d1) / np.maximum(d2, 1e-300)
    else:
        gap = np.full(N, np.inf)
    return AssignResult(labels.astype(np.int64), gap, d1, float(d1.sum()))


def update_centroids(X: np.ndarray, labels: np.ndarray, C_prev: np.ndarray) -> np.ndarray:
    """Alg. 1 'C <- Mean(X via L)' in raw token space.

    C_j = (1/|S_j|) sum_{i in S_j} x_i ; an empty cluster keeps its previous centroid (R5).
    """
    X = np.asarray(X, np.float64)
    C = np.array(C_prev, dtype=np.float64, copy=True)
    K = C.shape[0]
    for j in range(K):
        members = X[labels == j]
        if members.shape[0] > 0:
            C[j] = members.sum(axis=0) / members.shape[0]
    return C


@dataclass
class CoclusterResult:
    Lq: np.ndarray
    Cq: np.ndarray
    Lk: np.ndarray
    Ck: np.ndarray
    trace: list = field(default_factory=list)   # per half-step instrumentation


def cocluster(Q: np.ndarray, K: np.ndarray, kq: int, kk: int, iters: int, *,
              seed: int = 0, b: int = 0, h: int = 0, H: int = 1,
              init_q: np.ndarray | None = None, init_k: np.ndarray | None = None) -> CoclusterResult:
    """Algorithm 1, one (b, h) head (R6), literally.

    C_q^(0) <- Sample(Q, K_q); C_k^(0) <- Sample(K, K_k)
    for i = 1..I_max:
       Step A: L_k <- assign(K; anchors C_q^(i-1), self C_k^(i-1)); C_k^(i) <- Mean
       Step B: L_q <- assign(Q; anchors C_k^(i),   self C_q^(i-1)); C_q^(i) <- Mean
    return L_q, C_q, L_k, C_k  (R13: the post-update centroids)
    """
    if iters < 1:
        raise ValueError("I_max >= 1")
    Q = np.asarray(Q, np.float64)
    K = np.asarray(K, np.float64)
    N = Q.shape[0]
    if not (1 <= kq <= N and 1 <= kk <= K.shape[0]):
        raise ValueError("cluster counts must be in [1, N]")
    iq = init_q if init_q is not None else sample_anchor_indices(N, kq, seed, b, h, H, 0)
    ik = init_k if init_k is not None else sample_anchor_indices(K.shape[0], kk, seed, b, h, H, 1)
    Cq = Q[np.asarray(iq)].copy()
    Ck = K[np.asarray(ik)].copy()
    trace = []
    Lq = Lk = None
    for it in range(iters):
        ra = assign_step(K, Cq, Ck)               # Step A
        Ck_new = update_centroids(K, ra.labels, Ck)
        rb = assign_step(Q, Ck_new, Cq)           # Step B (uses C_k^(i) and C_q^(i-1))
        Cq_new = update_centroids(Q, rb.labels, Cq)
        trace.append(dict(it=it, side="k", labels=ra.labels, gap=ra.gap, C_anchor=Cq, C_self=Ck,
                          C_new=Ck_new, J=ra.objective))
        trace.append(dict(it=it, side="q", labels=rb.labels, gap=rb.gap, C_anchor=Ck_new, C_self=Cq,
                          C_new=Cq_new, J=rb.objective))
        Ck, Cq = Ck_new, Cq_new
        Lk, Lq = ra.labels, rb.labels
    return CoclusterResult(Lq, Cq, Lk, Ck, trace)


# ----------------------------------------------------------------------------------------------
# Independent k-means baseline ("w/o On" ablation; SVG2's partitioning, P:1270-1273;
# SURVEY §8f NEXT-2).  Queries and keys are clustered separately by Lloyd's algorithm in raw
# token space, initialised by the same sampler (R4).
# ----------------------------------------------------------------------------------------------
def kmeans_step(X: np.ndarray, C: np.ndarray) -> AssignResult:
    """L(i) = argmin_j ||x_i - c_j||_2 (ties -> lowest j); gap / objective as in assign_step."""
    X = np.asarray(X, np.float64)
    C = np.asarray(C, np.float64)
    sq = (X * X).sum(1)[:, None] + (C * C).sum(1)[None, :] - 2.0 * (X @ C.T)
    D = np.sqrt(np.maximum(sq, 0.0))
    labels = np.argmin(D, axis=1)
    N, K = D.shape
    d1 = D[np.arange(N), labels]
    if K > 1:
        D2 = D.copy()
        D2[np.arange(N), labels] = np.inf
        d2 = D2.min(axis=1)
        gap = (d2 - d1) / np.maximum(d2, 1e-300)
    else:
        gap = np.full(N, np.inf)
    return AssignResult(labels.astype(np.int64), gap, d1, float((d1 * d1).sum()))


def kmeans(X: np.ndarray, K: int, iters: int, *, seed: int = 0, b: int = 0, h: int = 0, H: int = 1,
           side: int = 0, init: np.ndarray | None = None):
    """Lloyd: C^(0) = X[Sample(X, K)] (R4, stream `side`); repeat iters times: assign, then
    C_j = mean of members (empty keeps its previous row, R5).  Returns (labels, C, trace) with the
    Lloyd objective sum_i ||x_i - c_L(i)||^2 of every assignment in trace."""
    X = np.asarray(X, np.float64)
    idx = init if init is not None else sample_anchor_indices(X.shape[0], K, seed, b, h, H, side)
    C = X[np.asarray(idx)].copy()
    trace = []
    labels = None
    for it in range(iters):
        r = kmeans_step(X, C)
        C_new = update_centroids(X, r.labels, C)
        trace.append(dict(it=it, labels=r.labels, gap=r.gap, C_self=C, C_new=C_new, J=r.objective))
        C, labels = C_new, r.labels
    return labels, C, trace


def cocluster_kmeans(Q: np.ndarray, K: np.ndarray, kq: int, kk: int, iters: int, *, seed: int = 0,
                     b: int = 0, h: int = 0, H: int = 1, init_q=None, init_k=None) -> CoclusterResult:
    """The "w/o On" partitioning: independent k-means of K (K_k clusters) and Q (K_q clusters),
    same sampler streams as Alg. 1 (keys side 1, queries side 0); same result type as cocluster."""
    Lk, Ck, tk = kmeans(K, kk, iters, seed=seed, b=b, h=h, H=H, side=1, init=init_k)
    Lq, Cq, tq = kmeans(Q, kq, iters, seed=seed, b=b, h=h, H=H, side=0, init=init_q)
    trace = []
    for a, c in zip(tk, tq):
        trace.append(dict(side="k", **a))
        trace.append(dict(side="q", **c))
    return CoclusterResult(Lq, Cq, Lk, Ck, trace)


# ----------------------------------------------------------------------------------------------
# Token permutation into contiguous clusters (implied by the dynamic block-size kernels)
# ----------------------------------------------------------------------------------------------
def counting_sort(labels: np.ndarray, K: int) -> tuple[np.ndarray, np.ndarray]:
    """Stable counting sort: histogram, exclusive scan, stable scatter.

    perm[p] = the token at sorted position p ; offs[c] .. offs[c+1] = the positions of cluster c.
    """
    labels = np.asarray(labels, np.int64)
    hist = [0] * K
    for c in labels:
        hist[int(c)] += 1
    offs = [0] * (K + 1)
    for c in range(K):
        offs[c + 1] = offs[c] + hist[c]
    pos = list(offs[:K])
    perm = [0] * len(labels)
    for i, c in enumerate(labels):
        perm[pos[int(c)]] = i
        pos[int(c)] += 1
    return np.array(perm, dtype=np.int64), np.array(offs, dtype=np.int64)


# ----------------------------------------------------------------------------------------------
# Top block-pair selection
# ----------------------------------------------------------------------------------------------
def n_from_ratio(r: float, Kk: int) -> int:
    """R10: a keep ratio r -> a block count: clamp(ceil(double(r)*K_k - 1e-3), 1, K_k)."""
    n = math.ceil(float(r) * Kk - 1e-3)
    return int(min(max(n, 1), Kk))


RECALL_EPS = 1e-12   # R9b: cumulative mass counts as reaching tau when cs >= tau - 1e-12


def recall_count(p_sorted: np.ndarray, tau: float) -> int:
    """R9: minimal prefix m of the descending masses whose sum reaches tau (R9b tolerance)."""
    cs = np.cumsum(np.asarray(p_sorted, np.float64))
    hit = np.nonzero(cs >= tau - RECALL_EPS)[0]
    return int(hit[0] + 1) if hit.size else int(len(cs))


def rule_count(n_rec: int, budget: float, theta: float, rule: int, Kk: int, Kk_ne: int) -> int:
    """The threshold-dependent rho rule in block counts (R8, R10).
    budget is a float32 per-head value (the ABI's budget array); theta and tau are doubles."""
    b = float(np.float32(budget))
    th = float(theta)
    n_b = n_from_ratio(b, Kk)
    if rule == RULE_DENSITY:
        n = min(n_rec, n_b) if (1.0 - b) > th else max(n_rec, n_b)
    elif rule == RULE_AS_WRITTEN:
        n = min(n_rec, n_b) if b > th else max(n_rec, n_b)
    elif rule == RULE_FIXED:
        n = n_b
    else:
        raise ValueError("rule")
    return int(min(max(n, 1), Kk_ne))


@dataclass
class SelectResult:
    n_keep: int
    kept: object            # [K_q, n_keep] ascending key-block indices (a list of per-row arrays
                            # when per_row: row a has n_rows[a] entries)
    c: np.ndarray           # per query block: minimal #key blocks covering tau (0 for empty rows)
    n_rec: int
    n_bud: int
    Abar: np.ndarray
    n_rows: np.ndarray | None = None  # per-row counts (per_row only)


def select_blocks(Cq: np.ndarray, Ck: np.ndarray, sizes_q: np.ndarray, sizes_k: np.ndarray,
                  budget: float, tau: float, theta: float, rule: int,
                  d_head: int | None = None, per_row: bool = False,
                  size_weighted: bool = False) -> SelectResult:
    """Coarse estimate, Recall, the threshold rule and top-rho K_k selection for one head.

    Abar = C_q C_k^T
    Recall(Abar, tau) (R9): for each nonempty query block a, p = softmax(Abar_a/sqrt(d)) over
        nonempty key blocks (R7); c_a = min{m : sum of the m largest p >= tau}; n_rec =
        ceil(sum_a c_a / K_q') (R10), K_q' = #nonempty query blocks; "reaches tau" is
        cs >= tau - 1e-12 (R9b) so exact-tie examples (uniform rows) are not decided by rounding.
    rho rule (R8):
        DENSITY    : budget b = d_hat (keep ratio); n = min(n_rec, n_b) if 1-b > theta else max(.)
        AS_WRITTEN : budget s = sparsity as printed; n = min(n_rec, n_s) if s > theta else max(.)
        FIXED      : n = n_b
    clamp n to [1, K_k'] ; kept[a] = the n key blocks with largest raw Abar_a (ties -> lowest
    index, empty key blocks never eligible), listed ascending (R11: same n every row).

    Variants of the readings R9 / R11 (R9c / R11b):
      size_weighted : block importance z_ac = Abar_ac / sqrt(d) + log|K_c| (the softmax mass of a
                      key block = the total attention mass its |K_c| tokens would get if each
                      had the centroid logit); ranking and Recall both use z (desc, index asc).
      per_row       : each nonempty query block a keeps n_a = rule(c_a) blocks — the same rho rule
                      with its own recall count c_a in place of the row mean n_rec; empty query
                      blocks keep the shared n.
    """
    Cq = np.asarray(Cq, np.float64)
    Ck = np.asarray(Ck, np.float64)
    Kq, d = Cq.shape
    Kk = Ck.shape[0]
    d_head = d if d_head is None else d_head
    A = Cq @ Ck.T
    ne_k = np.asarray(sizes_k) > 0
    ne_q = np.asarray(sizes_q) > 0
    Kk_ne = int(ne_k.sum())
    Kq_ne = int(ne_q.sum())
    cand = np.nonzero(ne_k)[0]
    orders = []
    c = np.zeros(Kq, dtype=np.int64)
    logsize = np.log(np.asarray(sizes_k, np.float64)[cand]) if size_weighted else None
    for a in range(Kq):
        if size_weighted:
            z = A[a, cand] / math.sqrt(d_head) + logsize
            o = cand[np.argsort(-z, kind="stable")]          # descending z, ties -> lower index
            zs = z[np.argsort(-z, kind="stable")]
        else:
            vals = A[a, cand]
            # descending raw Abar, ties -> lower index (stable sort on the negated values)
            o = cand[np.argsort(-vals, kind="stable")]
            zs = A[a, o] / math.sqrt(d_head)
        orders.append(o)
        if ne_q[a]:
            c[a] = recall_count(softmax_row(zs), float(tau))
    n_rec = (int(c.sum()) + Kq_ne - 1) // Kq_ne
    n_b = n_from_ratio(float(np.float32(budget)), Kk)
    n = rule_count(n_rec, budget, theta, rule, Kk, Kk_ne)
    if per_row:
        n_rows = np.array([rule_count(int(c[a]), budget, theta, rule, Kk, Kk_ne) if ne_q[a] else n
                           for a in range(Kq)], dtype=np.int64)
        kept = [np.sort(orders[a][:n_rows[a]]).astype(np.int64) for a in range(Kq)]
        return SelectResult(n, kept, c, n_rec, n_b, A, n_rows)
    kept = np.stack([np.sort(o[:n]) for o in orders]).astype(np.int64)
    return SelectResult(n, kept, c, n_rec, n_b, A)


# ----------------------------------------------------------------------------------------------
# Block-sparse attention and the dense ground truth
# ----------------------------------------------------------------------------------------------
def sparse_attention(Q, K, V, Lq, Lk, kept, scale: float | None = None) -> np.ndarray:
    """For query i in block a = L_q(i): allowed keys A_i = {j : L_k(j) in kept[a]};
    o_i = sum_{j in A_i} softmax_j(q_i.k_j * scale) v_j   (fp64, original token order)."""
    Q = np.asarray(Q, np.float64)
    K = np.asarray(K, np.float64)
    V = np.asarray(V, np.float64)
    N, d = Q.shape
    scale = 1.0 / math.sqrt(d) if scale is None else scale
    O = np.zeros((N, V.shape[1]))
    Lq = np.asarray(Lq)
    Lk = np.asarray(Lk)
    for a in np.unique(Lq):
        rows = np.nonzero(Lq == a)[0]
        allowed = np.nonzero(np.isin(Lk, np.asarray(kept[a])))[0]
        if allowed.size == 0:
            raise ValueError("empty allowed key set")
        S = (Q[rows] @ K[allowed].T) * scale
        S -= S.max(axis=1, keepdims=True)
        E = np.exp(S)
        O[rows] = (E @ V[allowed]) / E.sum(axis=1, keepdims=True)
    return O


def dense_attention(Q, K, V, scale: float | None = None) -> np.ndarray:
    """softmax(Q K^T * scale) V, fp64 (the rho = 1 ground truth)."""
    Q = np.asarray(Q, np.float64)
    K = np.asarray(K, np.float64)
    V = np.asarray(V, np.float64)
    scale = 1.0 / math.sqrt(Q.shape[1]) if scale is None else scale
    S = (Q @ K.T) * scale
    S -= S.max(axis=1, keepdims=True)
    E = np.exp(S)
    return (E @ V) / E.sum(axis=1, keepdims=True)


# ----------------------------------------------------------------------------------------------
# The whole layer, one head (north_star stages 1-5)
# ----------------------------------------------------------------------------------------------
@dataclass
class LayerResult:
    O: np.ndarray
    cc: CoclusterResult
    perm_q: np.ndarray
    offs_q: np.ndarray
    perm_k: np.ndarray
    offs_k: np.ndarray
    sel: SelectResult


def coclust_sparse_attention_head(Q, K, V, kq, kk, iters, seed, budget, tau, theta, rule,
                                  b=0, h=0, H=1, scale=None) -> LayerResult:
    cc = cocluster(Q, K, kq, kk, iters, seed=seed, b=b, h=h, H=H)
    perm_q, offs_q = counting_sort(cc.Lq, kq)
    perm_k, offs_k = counting_sort(cc.Lk, kk)
    sel = select_blocks(cc.Cq, cc.Ck, np.diff(offs_q), np.diff(offs_k), budget, tau, theta, rule,
                        d_head=np.asarray(Q).shape[1])
    O = sparse_attention(Q, K, V, cc.Lq, cc.Lk, sel.kept, scale)
    return LayerResult(O, cc, perm_q, offs_q, perm_k, offs_k, sel)


def kept_flops(offs_q: np.ndarray, offs_k: np.ndarray, kept: np.ndarray, d: int) -> int:
    """F_kept = sum_a 4 d |Q_a| sum_{c in kept[a]} |K_c|."""
    sq = np.diff(np.asarray(offs_q))
    sk = np.diff(np.asarray(offs_k))
    tot = 0
    for a in range(len(sq)):
        tot += int(sq[a]) * int(sk[np.asarray(kept[a])].sum())
    return 4 * d * tot


# ----------------------------------------------------------------------------------------------
# Matched-budget attention recall (R19)
# ----------------------------------------------------------------------------------------------
def reference_pairs(A: np.ndarray, mass: float = 0.5) -> np.ndarray:
    """The high-attention reference set: sort all token pairs by A_ij (desc) and take the
    smallest prefix whose cumulative attention mass reaches `mass` of the total.  Returns a
    boolean [N, N] mask.  A is the dense attention matrix (rows sum to 1)."""
    A = np.asarray(A, np.float64)
    flat = A.ravel()
    order = np.argsort(-flat, kind="stable")
    cs = np.cumsum(flat[order])
    m = int(np.searchsorted(cs, mass * cs[-1], side="left")) + 1
    mask = np.zeros(flat.shape, dtype=bool)
    mask[order[:m]] = True
    return mask.reshape(A.shape)


def block_pair_counts(ref: np.ndarray, Lq: np.ndarray, Lk: np.ndarray, kq: int, kk: int) -> np.ndarray:
    """cnt[a, c] = #{(i, j) in ref : L_q(i) = a, L_k(j) = c}: reference pairs covered by the block
    pair (a, c) ("a token pair is covered if its query token and key token fall into the
    selected Q-K block pair")."""
    cnt = np.zeros((kq, kk), dtype=np.int64)
    ii, jj = np.nonzero(ref)
    np.add.at(cnt, (np.asarray(Lq)[ii], np.asarray(Lk)[jj]), 1)
    return cnt


def block_pair_recall(cnt: np.ndarray, budget_pairs: int) -> float:
    """Recall of the reference set with `budget_pairs` block pairs, each method choosing its best
    pairs (most covered reference pairs first, ties -> lowest flat index)."""
    flat = cnt.ravel()
    order = np.argsort(-flat, kind="stable")
    tot = int(flat.sum())
    return float(flat[order[:budget_pairs]].sum()) / tot if tot else 1.0


def pairs_to_cover(cnt: np.ndarray, frac: float = 1.0) -> int:
    """Fewest block pairs whose covered reference pairs reach `frac` of the reference set."""
    flat = np.sort(cnt.ravel())[::-1]
    cs = np.cumsum(flat)
    return int(np.searchsorted(cs, frac * cs[-1] - 1e-9, side="left")) + 1


# ----------------------------------------------------------------------------------------------
# Offline layer-wise sparsity profiling
# ----------------------------------------------------------------------------------------------
def attention_density(A: np.ndarray, tau: float = 0.95) -> tuple[float, np.ndarray]:
    """for each row i of the post-softmax attention A (n x n), S(i) = the minimal
    descending prefix with sum >= tau ("reaches tau" with the R9b tolerance 1e-12);
    d = (1/n) sum_i |S(i)| / n.  Returns (d, |S(i)| per row)."""
    A = np.asarray(A, np.float64)
    n = A.shape[1]
    counts = np.empty(A.shape[0], dtype=np.int64)
    for i in range(A.shape[0]):
        cs = np.cumsum(np.sort(A[i])[::-1])
        hit = np.nonzero(cs >= tau - RECALL_EPS)[0]
        counts[i] = hit[0] + 1 if hit.size else n
    return float(counts.sum()) / A.shape[0] / n, counts


def attention_density_qk(Q: np.ndarray, K: np.ndarray, tau: float = 0.95, scale: float | None = None):
    """attention_density of A = softmax(Q K^T * scale) (rows), fp64 (one head)."""
    Q = np.asarray(Q, np.float64)
    K = np.asarray(K, np.float64)
    scale = 1.0 / math.sqrt(Q.shape[1]) if scale is None else scale
    S = Q @ K.T * scale
    S -= S.max(1, keepdims=True)
    E = np.exp(S)
    return attention_density(E / E.sum(1, keepdims=True), tau)


Z_95 = 1.6448536269514722   # upper 0.95 quantile of N(0, 1) (alpha = 0.95)


def sparsity_schedule(d: np.ndarray, z: float = Z_95) -> dict:
    """fit N(mu, sigma^2) to the m calibration densities of each (layer, head)
    (axis 0 of d: [m, L, H]; maximum-likelihood sigma), d_hat = mu + z_alpha sigma, s = 1 - d_hat.
    d_hat is clamped to 1 (R21: a density cannot exceed 1); it is the keep budget the DENSITY rule
    consumes (R8)."""
    d = np.asarray(d, np.float64)
    mu = d.mean(axis=0)
    sigma = d.std(axis=0, ddof=0)
    d_hat = np.minimum(mu + z * sigma, 1.0)
    return {"mu": mu, "sigma": sigma, "d_hat": d_hat, "s": 1.0 - d_hat}
