/*
 * coclust.h — C ABI of libcoclust.so, the B200 (sm_100a) hot path of SVOO (arXiv 2603.18636):
 * per-head online bidirectional co-clustering of queries and keys, cluster permutation,
 * centroid-level block selection under a per-layer keep budget, and varlen block-sparse flash
 * attention with the inverse permutation fused into its stores.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n (Alg. 1 = P:1203-1229, selection = P:1247-1257,
 * kernels = P:1266); R1..R17 = the readings listed in DESIGN.md ("Readings of the paper").
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 * - Every pointer argument is a DEVICE pointer owned by the caller (the library never allocates,
 *   frees or synchronises).  `stream` is a cudaStream_t passed as void*; every call only enqueues
 *   work on it.  Calls are reentrant: no global mutable state.
 * - Q, K, V, O are bf16 [B, H, N, d] given as (ptr, sb, sh, sn): element strides of the B, H and N
 *   dimensions; the d dimension must be contiguous (stride 1).  Both [B,H,N,d] and [B,N,H,d]
 *   buffers are expressible.  d must be 64 or 128.  ptr must be 16-byte aligned and sb, sh, sn
 *   multiples of 8 elements (TMA); broadcast views (stride 0 over an extent > 1) and overlapping
 *   rows (sn < d with N > 1) are rejected with CS_ERR_SHAPE.
 * - "bh" below is b*H + h.  Labels are int32 in [0, k).  perm[bh][p] = the token at cluster-sorted
 *   position p (stable: ascending token index inside a cluster); offs[bh][c]..offs[bh][c+1] are the
 *   positions of cluster c (offs[bh][0] = 0, offs[bh][k] = N).
 * - Centroids are fp32 [B, H, k, d] contiguous.
 * - ws / ws_bytes: caller-owned scratch of at least cs_workspace_bytes(...) bytes, 16-byte
 *   aligned (CS_ERR_ALIGN otherwise; the library rounds the base up to 256 bytes inside the
 *   slack cs_workspace_bytes includes).  Its contents are undefined between calls.
 * - Errors: arguments are validated on the host BEFORE anything is enqueued; on error nothing is
 *   launched and a cs_status != CS_OK is returned; cs_last_error() (thread-local) holds a message.
 *   CS_ERR_CUDA reports a launch error; asynchronous device faults surface at the caller's next
 *   synchronisation, as usual for CUDA.
 * - Results are deterministic (no floating-point atomics) and independent of how many heads or
 *   GPUs share a launch.
 */
#ifndef COCLUST_H
#define COCLUST_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  CS_OK = 0,
  CS_ERR_NULL = 1,        /* a required pointer is NULL                                       */
  CS_ERR_SHAPE = 2,       /* B,H,N <= 0, d not in {64,128}, inconsistent strides: a stride of 0
                             on a dimension of extent > 1 (broadcast) or sn < d (overlapping rows) */
  CS_ERR_ARG = 3,         /* k > N or k > 1024, iters < 1, tau not in (0,1], theta not in (0,1),
                             scale <= 0, unknown rule                                           */
  CS_ERR_ALIGN = 4,       /* pointer not 16-byte aligned or stride not a multiple of 8 elements */
  CS_ERR_WORKSPACE = 5,   /* ws NULL or smaller than required                                  */
  CS_ERR_UNSUPPORTED = 6, /* a size the kernels do not handle (e.g. N >= 2^24)                 */
  CS_ERR_CUDA = 7         /* a CUDA launch / driver call failed                                */
} cs_status;

typedef struct { const void* ptr; int64_t sb, sh, sn; } cs_bf16_in;
typedef struct { void* ptr; int64_t sb, sh, sn; } cs_bf16_out;

/* The threshold-dependent rho rule, read per R8:
 *   CS_RULE_DENSITY    budget[h] = d_hat (keep ratio):  n = min(n_rec, n_b) if 1-b > theta else max
 *   CS_RULE_AS_WRITTEN budget[h] = s (sparsity, literal): n = min(n_rec, n_s) if s > theta else max
 *   CS_RULE_FIXED      n = n_b (keep-ratio sweeps)
 * with n_b = clamp(ceil(double(b)*k_k - 1e-3), 1, k_k) (R10), n_rec from Recall (R9), and the
 * result clamped to [1, #nonempty key clusters].                                                 */
typedef enum { CS_RULE_DENSITY = 0, CS_RULE_AS_WRITTEN = 1, CS_RULE_FIXED = 2 } cs_rule;

/* Library version (major*10000 + minor*100 + patch). */
int cs_version(void);
/* Static text for a status code. */
const char* cs_status_string(int status);
/* Thread-local detail of the last error returned on this thread ("" if none). */
const char* cs_last_error(void);

/* Scratch bytes needed by any entry point below for these sizes (the maximum over entries). */
size_t cs_workspace_bytes(int B, int H, int N, int d, int kq, int kk);

/* ---------------------------------------------------------------------------------------------
 * coclust_assign — Algorithm 1 for every (b,h), then the cluster permutation.
 *   C_q^(0) = Q[Sample(N,kq)], C_k^(0) = K[Sample(N,kk)] (R4: Floyd sampling over splitmix64 with
 *   stream seed seed ^ (((b*Ht+hg)*2+side) * 0x9E3779B97F4A7C15), side 0 = Q, 1 = K, where
 *   hg = head_offset + h is the global head index and Ht = heads_total (0 -> H, head_offset must
 *   then be 0) — so a head-sharded call reproduces the single-call streams bit for bit;
 *   explicit index arrays init_q [B,H,kq] / init_k [B,H,kk] override the sampler when non-NULL);
 *   iters times: Step A (keys; anchors C_q, self C_k) then Step B (queries; anchors the
 *   new C_k, self the old C_q).  Assignment = argmin of the Euclidean distance
 *   between L2-normalised affinity rows (R1-R3), evaluated in the exact reduced form
 *   argmax_j x.W_j; ties -> lowest j.  Mean update in raw token space;
 *   an empty cluster keeps its previous centroid (R5).
 * Outputs: cq [B,H,kq,d], ck [B,H,kk,d] fp32 (post-update, R13); lq, lk int32 [B,H,N];
 *   perm_q, perm_k int32 [B,H,N]; offs_q int32 [B,H,kq+1]; offs_k int32 [B,H,kk+1]. */
cs_status coclust_assign(int B, int H, int N, int d, cs_bf16_in q, cs_bf16_in k, int kq, int kk,
                         int iters, uint64_t seed, int head_offset, int heads_total,
                         const int32_t* init_q, const int32_t* init_k,
                         float* cq, float* ck, int32_t* lq, int32_t* lk, int32_t* perm_q,
                         int32_t* offs_q, int32_t* perm_k, int32_t* offs_k, void* ws,
                         size_t ws_bytes, void* stream);

/* One assignment half-step of Alg. 1 with given centroids (parity helper):
 * x [B,H,N,d] bf16; c_anchor [B,H,ka,d] fp32 (the other side's centroids); c_self [B,H,ks,d] fp32;
 * labels out int32 [B,H,N].  ka, ks in [1,1024]. */
cs_status coclust_assign_step(int B, int H, int N, int d, cs_bf16_in x, int ka,
                              const float* c_anchor, int ks, const float* c_self,
                              int32_t* labels, void* ws, size_t ws_bytes, void* stream);

/* Independent k-means baseline (the "w/o On" ablation; SVG2's K-means partitioning,
 * P:1270-1273).  Same arguments, outputs and sampler (R4) as coclust_assign, but
 * each side is clustered alone by Lloyd's algorithm in raw token space: L(i) = argmin_j
 * ||x_i - c_j||_2 (ties -> lowest j), then C_j = member mean (empty keeps its row, R5); keys
 * first, then queries, iters times.  Computed by the assignment GEMM with W_j = c_j (bf16 hi + lo)
 * and a -||c_j||^2/2 bias in the argmax epilogue. */
cs_status kmeans_assign(int B, int H, int N, int d, cs_bf16_in q, cs_bf16_in k, int kq, int kk,
                        int iters, uint64_t seed, int head_offset, int heads_total,
                        const int32_t* init_q, const int32_t* init_k, float* cq, float* ck,
                        int32_t* lq, int32_t* lk, int32_t* perm_q, int32_t* offs_q, int32_t* perm_k,
                        int32_t* offs_k, void* ws, size_t ws_bytes, void* stream);

/* One k-means assignment with given centroids c_self [B,H,ks,d] fp32 -> labels [B,H,N] (parity
 * helper, as coclust_assign_step). */
cs_status kmeans_assign_step(int B, int H, int N, int d, cs_bf16_in x, int ks, const float* c_self,
                             int32_t* labels, void* ws, size_t ws_bytes, void* stream);

/* Centroid update "C <- Mean(X via L)": c_inout [B,H,k,d] fp32; rows of empty clusters
 * are left unchanged (R5).  perm/offs as produced by coclust_permute.  If x_perm is non-NULL it
 * also receives the cluster-sorted copy x_perm[bh][p][:] = x[b,h,perm[bh][p],:] (bf16,
 * [B*H, N, d] contiguous). */
cs_status coclust_update_centroids(int B, int H, int N, int d, cs_bf16_in x, int k,
                                   const int32_t* perm, const int32_t* offs, float* c_inout,
                                   void* x_perm, void* stream);

/* Stable counting sort of labels [BH, N] into perm [BH, N] and offs [BH, k+1] (implied by the
 * dynamic block-size kernels). */
cs_status coclust_permute(int BH, int N, int k, const int32_t* labels, int32_t* perm,
                          int32_t* offs, void* ws, size_t ws_bytes, void* stream);

/* Top block-pair selection per (b,h):
 *   Abar = C_q C_k^T in fp64 (columns of empty key clusters excluded, R9);
 *   for each nonempty query block a: p = softmax(Abar_a / sqrt(d)) (R7),
 *   c_a = min{m : sum of the m largest p >= tau - 1e-12} (R9, R9b), n_rec = ceil(sum c_a / Kq');
 *   n from the rule (cs_rule, budget[h] float32, theta); kept[b][h][a][0..n) = the n key clusters
 *   with largest raw Abar_a (ties -> lower index), ascending.  Entries past n are not written.
 * budget [H] float32; tau in (0,1]; theta in (0,1).  n_keep out int32 [B,H]; kept out int32
 * [B,H,kq,kk]. */
cs_status block_select(int B, int H, int kq, int kk, int d, const float* cq, const float* ck,
                       const int32_t* offs_q, const int32_t* offs_k, const float* budget,
                       double tau, double theta, int rule, int32_t* n_keep, int32_t* kept,
                       void* ws, size_t ws_bytes, void* stream);

/* Selection variants (the paper's Recall and "top rho K_k" are open to these
 * readings, R9c / R11b).  Bit flags: */
enum {
  /* R11b: each nonempty query block a keeps n_a = rule(c_a) blocks (the same rho rule with its
   * own recall count in place of the row mean n_rec); empty query blocks keep the shared n. */
  CS_SEL_PER_ROW = 1,
  /* R9c: block importance z_ac = Abar_ac / sqrt(d) + log|K_c| (softmax mass of a key block =
   * the mass its |K_c| tokens would get at the centroid logit); ranking and Recall both use z
   * (descending, ties -> lower index). */
  CS_SEL_SIZE_WEIGHTED = 2,
  /* Fused entries only: partition Q and K by the independent k-means baseline (kmeans_assign)
   * instead of Alg. 1 co-clustering — the paper's "w/o On" ablation, SVG2-style. */
  CS_CLUSTER_KMEANS = 0x100
};

/* block_select with selection flags.  n_keep [B,H] always receives the shared count (R11);
 * n_keep_rows [B,H,kq] (required with CS_SEL_PER_ROW, else nullable) receives the per-row counts
 * (the shared n in every row without CS_SEL_PER_ROW); kept row a holds n_keep_rows[a] ascending
 * entries.  Unknown flag bits -> CS_ERR_ARG. */
cs_status block_select_ex(int B, int H, int kq, int kk, int d, const float* cq, const float* ck,
                          const int32_t* offs_q, const int32_t* offs_k, const float* budget,
                          double tau, double theta, int rule, int flags, int32_t* n_keep,
                          int32_t* n_keep_rows, int32_t* kept, void* ws, size_t ws_bytes,
                          void* stream);

/* Block-sparse attention over the kept blocks.
 *   for query i in cluster a: o_i = sum_{j: L_k(j) in kept[a]} softmax_j(q_i.k_j * scale) v_j,
 * written in ORIGINAL token order (the inverse permutation is fused into the stores).  bf16 MMA,
 * fp32 accumulation and softmax, bf16 P (R15).  scale > 0 (1/sqrt(d) for the paper).
 * A caller-supplied kept row whose clusters are all empty (no allowed key: the softmax over an
 * empty set, S:419's contract violation) gives o_i = 0 for the queries of that row; block_select
 * never produces such a row (n_keep >= 1 over nonempty key clusters only). */
cs_status block_sparse_attn(int B, int H, int N, int d, cs_bf16_in q, cs_bf16_in k, cs_bf16_in v,
                            int kq, int kk, const int32_t* perm_q, const int32_t* offs_q,
                            const int32_t* perm_k, const int32_t* offs_k, const int32_t* n_keep,
                            const int32_t* kept, float scale, cs_bf16_out o, void* ws,
                            size_t ws_bytes, void* stream);

/* block_sparse_attn with per-row kept counts: n_keep_rows [B,H,kq] (nullable -> n_keep[b,h] for
 * every row), as written by block_select_ex. */
cs_status block_sparse_attn_ex(int B, int H, int N, int d, cs_bf16_in q, cs_bf16_in k, cs_bf16_in v,
                               int kq, int kk, const int32_t* perm_q, const int32_t* offs_q,
                               const int32_t* perm_k, const int32_t* offs_k, const int32_t* n_keep,
                               const int32_t* n_keep_rows, const int32_t* kept, float scale,
                               cs_bf16_out o, void* ws, size_t ws_bytes, void* stream);

/* The whole layer: coclust_assign -> block_select -> block_sparse_attn, on device only (no host
 * round trip; CUDA-graph capturable).  budget [H] is indexed by the local head h; head_offset /
 * heads_total as in coclust_assign.  stage_events (nullable) = 4 cudaEvent_t recorded on `stream`
 * (0) after co-clustering, (1) after block selection, (2) just before and (3) just after the
 * block-sparse attention kernel — for per-stage timing by the caller. */
cs_status coclust_sparse_attention(int B, int H, int N, int d, cs_bf16_in q, cs_bf16_in k,
                                   cs_bf16_in v, int kq, int kk, int iters, uint64_t seed,
                                   int head_offset, int heads_total,
                                   const float* budget, double tau, double theta, int rule,
                                   float scale, cs_bf16_out o, void* ws, size_t ws_bytes,
                                   void* stream, void* const* stage_events);

/* coclust_sparse_attention with flags (CS_SEL_* selection variants, CS_CLUSTER_KMEANS baseline
 * partitioning); sel_flags = 0 is the base entry. */
cs_status coclust_sparse_attention_ex(int B, int H, int N, int d, cs_bf16_in q, cs_bf16_in k,
                                      cs_bf16_in v, int kq, int kk, int iters, uint64_t seed,
                                      int head_offset, int heads_total, const float* budget,
                                      double tau, double theta, int rule, int sel_flags,
                                      float scale, cs_bf16_out o, void* ws, size_t ws_bytes,
                                      void* stream, void* const* stage_events);

/* Clustering-reuse state ("we reuse the clustering results and recompute them every
 * N steps").  Caller-owned device buffers, shapes as in coclust_assign /
 * block_select. */
typedef struct {
  float* cq;       /* [B,H,kq,d] */
  float* ck;       /* [B,H,kk,d] */
  int32_t* lq;     /* [B,H,N]    */
  int32_t* lk;     /* [B,H,N]    */
  int32_t* perm_q; /* [B,H,N]    */
  int32_t* perm_k; /* [B,H,N]    */
  int32_t* offs_q; /* [B,H,kq+1] */
  int32_t* offs_k; /* [B,H,kk+1] */
  int32_t* n_keep; /* [B,H]      */
  int32_t* kept;   /* [B,H,kq,kk]*/
  int32_t* n_keep_rows; /* [B,H,kq] per-row counts; NULL allowed unless sel_flags has CS_SEL_PER_ROW */
} cs_layer_state;

/* coclust_sparse_attention with caller-owned state: recompute != 0 runs co-clustering and selection
 * and stores them in *state; recompute == 0 skips both and reuses *state (only Q, K, V are
 * re-permuted), so a caller recomputes every R_reuse denoising steps (R14). */
cs_status coclust_sparse_attention_cached(int B, int H, int N, int d, cs_bf16_in q, cs_bf16_in k,
                                          cs_bf16_in v, int kq, int kk, int iters, uint64_t seed,
                                          int head_offset, int heads_total, const float* budget,
                                          double tau, double theta, int rule, int sel_flags,
                                          float scale, cs_bf16_out o, const cs_layer_state* state,
                                          int recompute,
                                          void* ws, size_t ws_bytes, void* stream,
                                          void* const* stage_events);

/* Offline layer-wise sparsity profiling.  For every (b,h):
 *   A = softmax(q k^T * scale) (rows), S(i) = the minimal descending prefix of row i whose mass
 *   reaches tau (R9b tolerance 1e-12), counts[b][h][i] = |S(i)| (nullable [B,H,N] int32 out),
 *   density[b][h] = (1/N) sum_i |S(i)| / N (double out [B,H]).
 * No sort: after a row max / row sum pass, `passes` (0 -> 4, at most 5) radix passes over the float
 * bits of p = 2^(logit - max) (exponent, then 5 mantissa bits per pass) locate the crossing of the
 * descending cumulative mass to p-values sharing exponent and 5 (passes-1) mantissa bits; the
 * count inside that final bin is interpolated from its elements' mean mass (exact unless several
 * elements share the bin).  Each pass recomputes Q K^T on the tensor cores.  The Gaussian fit over
 * calibration inputs and the schedule s = 1 - d_hat are host-side
 * (paper_2603_18636_b200/profiler.py).  Workspace: cs_density_workspace_bytes(B, H, N). */
size_t cs_density_workspace_bytes(int B, int H, int N);
cs_status attention_density(int B, int H, int N, int d, cs_bf16_in q, cs_bf16_in k, double tau,
                            float scale, int passes, int32_t* counts, double* density, void* ws,
                            size_t ws_bytes, void* stream);

/* ---- Fused Ulysses return path: the attention epilogue stores each output row
 * straight into the token block of the rank that owns the token (NVLink P2P / CUDA IPC mapped
 * pointers), fusing the inverse permutation AND the return all-to-all into the attention kernel.
 * Rank p's output block is [N/P, H_total, d] bf16 with element strides s_tok (token) and s_head
 * (head), d contiguous; token n of this call goes to rank n / n_per_rank, row n % n_per_rank,
 * head head_base + h. */
typedef struct {
  const void* ptrs;    /* DEVICE array of P uint64 device pointers (peer blocks mapped here) */
  int P;               /* ranks; P * n_per_rank == N */
  int n_per_rank;
  int head_base;       /* global head index of this call's head 0 */
  int64_t s_tok, s_head;
} cs_peer_out;

/* coclust_sparse_attention (B = 1) with its output scattered to the peers' token blocks.  The
 * caller orders the consumers after all ranks' calls, e.g. with cs_peer_barrier on the stream. */
cs_status coclust_sparse_attention_peer(int H, int N, int d, cs_bf16_in q, cs_bf16_in k,
                                        cs_bf16_in v, int kq, int kk, int iters, uint64_t seed,
                                        int head_offset, int heads_total, const float* budget,
                                        double tau, double theta, int rule, int flags, float scale,
                                        const cs_peer_out* o, void* ws, size_t ws_bytes,
                                        void* stream, void* const* stage_events);

/* The Ulysses layer entry (B = 1): coclust_sparse_attention_ex on the [1, H, N, d]
 * strided views of the in-bound all-to-all buffers, with two multi-GPU hooks:
 *   v_ready  (nullable cudaEvent_t) — `stream` waits on it just before V is first read, after
 *            co-clustering and selection (which read only Q and K): the caller's all-to-all of V
 *            on another stream overlaps the whole clustering stage;
 *   peer     (nullable) — output rows go to the owners' token blocks as in
 *            coclust_sparse_attention_peer; o is ignored then.  Otherwise o receives the output. */
cs_status coclust_sparse_attention_ulysses(int H, int N, int d, cs_bf16_in q, cs_bf16_in k,
                                           cs_bf16_in v, int kq, int kk, int iters, uint64_t seed,
                                           int head_offset, int heads_total, const float* budget,
                                           double tau, double theta, int rule, int flags, float scale,
                                           cs_bf16_out o, const cs_peer_out* peer, void* v_ready,
                                           void* ws, size_t ws_bytes, void* stream,
                                           void* const* stage_events);

/* Ulysses in-bound pack (a13): T (1..4) rank-local token blocks srcs[t] = [Nl, P*Hl, d] bf16
 * (host array of T device pointers, 16-byte aligned) -> dst [P, Nl, T, Hl, d]: chunk p holds the
 * heads of rank p, and per token the T tensors' head rows side by side.  After one
 * all_to_all_single of dst the receiver holds [N = P*Nl, T, Hl, d], in which tensor t is the
 * [1, Hl, N, d] view with element strides (sh, sn) = (d, T*Hl*d) — passed to the layer as is. */
cs_status cs_ulysses_pack(int Nl, int P, int Hl, int d, int T, const void* const* srcs, void* dst,
                          void* stream);

/* Head-group form of cs_ulysses_pack (the in-bound exchange split by head groups, so
 * group g+1's all_to_all overlaps group g's layer): packs only heads [g*Hg, (g+1)*Hg) of every
 * rank's Hl-head block, dst [P, Nl, T, Hg, d]; after the all_to_all_single tensor t is the
 * [1, Hg, N, d] view with strides (d, T*Hg*d) of the receive buffer.  Hg must divide Hl,
 * 0 <= g < Hl/Hg; cs_ulysses_pack is the case Hg = Hl, g = 0.  Same pointer rules; CS_ERR_ARG on a
 * bad group. */
cs_status cs_ulysses_pack_group(int Nl, int P, int Hl, int Hg, int g, int d, int T, const void* const* srcs,
                                void* dst, void* stream);

/* Device-side barrier over P ranks: peer_flags = DEVICE array of P uint64 pointers to every
 * rank's int32 flag array [P] (zero-initialised, mapped here); rank `rank` writes `epoch` into
 * flags_p[rank] of every rank p (system-scope release) after all earlier work on `stream`, then
 * waits until its own flags[p] >= epoch for all p (acquire).  epoch >= 1, increasing per use.
 * A peer that never arrives makes the kernel trap after ~2^32 cycles (launch error, no hang). */
cs_status cs_peer_barrier(int P, int rank, const void* peer_flags, int epoch, void* stream);

/* CUDA IPC export / import of caller-owned device memory: handle_out receives the 64-byte
 * cudaIpcMemHandle of the allocation containing dev_ptr and offset_out dev_ptr's offset in it;
 * cs_ipc_open maps a peer's handle (lazy peer access) and returns the peer pointer (base +
 * offset); cs_ipc_close unmaps it. */
cs_status cs_ipc_handle(const void* dev_ptr, void* handle_out, size_t* offset_out);
cs_status cs_ipc_open(const void* handle, size_t offset, void** dev_ptr_out);
cs_status cs_ipc_close(void* dev_ptr, size_t offset);

/* Ulysses resharding helper (BASELINE configs[3]): dst[b][a] = src[a][b] for an
 * [A, B] grid of rows of row_bytes bytes (row_bytes a multiple of 16, pointers 16-byte aligned).
 * Packs a [N/P, H, d] token block into [P, N/P, H/P, d] per-destination chunks before the
 * all-to-all (A = N/P, B = P, row = H/P*d) and unpacks the returned chunks after it. */
cs_status cs_block_transpose(int A, int B, size_t row_bytes, const void* src, void* dst, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* COCLUST_H */
