// api.cu — the C ABI of libcoclust.so (include/coclust.h): host-side validation, workspace
// carving, TMA descriptor encoding and the launch sequences.  No entry point allocates, frees or
// synchronises; every launch goes to the caller's stream.
#include <cuda.h>
#include <nvtx3/nvToolsExt.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <mutex>

#include "../../include/coclust.h"
#include "kernels.cuh"

using namespace cs;

namespace {

thread_local char g_err[512] = "";

cs_status fail(cs_status s, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return s;
}
cs_status cuda_fail(cudaError_t e, const char* where) {
  return fail(CS_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}
#define CS_CUDA(call, where)                          \
  do {                                                \
    cudaError_t _e = (call);                          \
    if (_e != cudaSuccess) return cuda_fail(_e, where); \
  } while (0)
#define CS_CHECK(expr)             \
  do {                             \
    cs_status _s = (expr);         \
    if (_s != CS_OK) return _s;    \
  } while (0)

// NVTX ranges around the host-side enqueue of each stage (SURVEY §5 per-stage markers: visible to
// nsys / `ncu --nvtx --nvtx-include`); header-only NVTX3, a no-op unless a tool is attached.
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
};

// ---------------------------------------------------------------- workspace carving
struct Carve {
  uint8_t* base;  // nullptr -> sizing pass
  size_t off = 0;
  // the base is rounded up to 256 bytes (every need_* adds 256 bytes of slack for this), so a
  // 16-byte-aligned caller workspace still gives 256-byte-aligned scratch arrays
  explicit Carve(void* b)
      : base(b ? reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(b) + 255) & ~uintptr_t(255)) : nullptr) {}
  template <typename T>
  T* take(size_t count) {
    off = (off + 255) & ~size_t(255);
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += count * sizeof(T);
    return p;
  }
};

int round_up(int x, int m) { return (x + m - 1) / m * m; }
int chunk_n(int ks) { return assign_chunk_n(ks); }
int pad_k(int ks) {
  const int n = chunk_n(ks);
  return (ks + n - 1) / n * n;
}

struct AssignScratch {
  double* gamma;
  __nv_bfloat16* wsplit;
  int32_t* hist;
  float* bias;  // k-means baseline: -||c_j||^2 / 2 per (bh, padded centroid)
};
AssignScratch carve_assign(Carve& c, int BH, int N, int d, int kq, int kk) {
  AssignScratch s;
  const int kmax = std::max(kq, kk);
  // partial Gammas of the anchor-row splits (k_gamma): ceil(K_a / kGammaRows) slabs
  s.gamma = c.take<double>((size_t)((kmax + kGammaRows - 1) / kGammaRows) * BH * d * d);
  s.wsplit = c.take<__nv_bfloat16>((size_t)BH * std::max(pad_k(kq), pad_k(kk)) * 2 * d);
  s.hist = c.take<int32_t>((size_t)BH * ((N + kSortTile - 1) / kSortTile + 1) * kmax);  // + label sizes
  s.bias = c.take<float>((size_t)BH * std::max(pad_k(kq), pad_k(kk)));
  return s;
}
struct SelectScratch {
  int32_t* order;
  int32_t* cnt;
  double* abar;
};
SelectScratch carve_select(Carve& c, int BH, int kq, int kk) {
  SelectScratch s;
  s.order = c.take<int32_t>((size_t)BH * kq * kk);
  s.cnt = c.take<int32_t>((size_t)BH * kq);
  s.abar = c.take<double>((size_t)BH * kq * kk);
  return s;
}
struct AttnScratch {
  __nv_bfloat16 *qp, *kp, *vp;
  int32_t* item_start;
};
AttnScratch carve_attn(Carve& c, int BH, int N, int d, int kq) {
  AttnScratch s;
  s.qp = c.take<__nv_bfloat16>((size_t)BH * N * d);
  s.kp = c.take<__nv_bfloat16>((size_t)BH * N * d);
  s.vp = c.take<__nv_bfloat16>((size_t)BH * N * d);
  s.item_start = c.take<int32_t>((size_t)BH * (kq + 1));
  return s;
}
struct LayerState {
  float *cq, *ck;
  int32_t *lq, *lk, *perm_q, *perm_k, *offs_q, *offs_k, *n_keep, *kept;
  int32_t* n_rows;  // per-row kept counts [BH, kq] (nullable in the cached entry: shared n only)
};
LayerState carve_state(Carve& c, int BH, int N, int d, int kq, int kk) {
  LayerState s;
  s.cq = c.take<float>((size_t)BH * kq * d);
  s.ck = c.take<float>((size_t)BH * kk * d);
  s.lq = c.take<int32_t>((size_t)BH * N);
  s.lk = c.take<int32_t>((size_t)BH * N);
  s.perm_q = c.take<int32_t>((size_t)BH * N);
  s.perm_k = c.take<int32_t>((size_t)BH * N);
  s.offs_q = c.take<int32_t>((size_t)BH * (kq + 1));
  s.offs_k = c.take<int32_t>((size_t)BH * (kk + 1));
  s.n_keep = c.take<int32_t>((size_t)BH);
  s.kept = c.take<int32_t>((size_t)BH * kq * kk);
  s.n_rows = c.take<int32_t>((size_t)BH * kq);
  return s;
}

size_t need_assign(int BH, int N, int d, int kq, int kk) {
  Carve c(nullptr);
  carve_assign(c, BH, N, d, kq, kk);
  return c.off + 256;
}
size_t need_select(int BH, int kq, int kk) {
  Carve c(nullptr);
  carve_select(c, BH, kq, kk);
  return c.off + 256;
}
size_t need_attn(int BH, int N, int d, int kq) {
  Carve c(nullptr);
  carve_attn(c, BH, N, d, kq);
  return c.off + 256;
}
size_t need_layer(int BH, int N, int d, int kq, int kk) {
  Carve c(nullptr);
  carve_state(c, BH, N, d, kq, kk);
  carve_attn(c, BH, N, d, kq);
  carve_assign(c, BH, N, d, kq, kk);
  carve_select(c, BH, kq, kk);
  return c.off + 256;
}

// ---------------------------------------------------------------- validation
cs_status check_dims(int B, int H, int N, int d) {
  if (B <= 0 || H <= 0 || N <= 0) return fail(CS_ERR_SHAPE, "B, H, N must be positive (got %d, %d, %d)", B, H, N);
  if (d != 64 && d != 128) return fail(CS_ERR_SHAPE, "d must be 64 or 128 (got %d)", d);
  if (N >= (1 << 24)) return fail(CS_ERR_UNSUPPORTED, "N must be < 2^24 (got %d)", N);
  if ((long long)B * H * N >= (1LL << 31)) return fail(CS_ERR_UNSUPPORTED, "B*H*N must be < 2^31");
  return CS_OK;
}
cs_status check_k(int k, int N, const char* name) {
  if (k < 1 || k > N || k > kMaxClusters)
    return fail(CS_ERR_ARG, "%s must be in [1, min(N, %d)] (got %d, N=%d)", name, kMaxClusters, k, N);
  return CS_OK;
}
// A [B, H, N, d] bf16 operand: 16-byte aligned, strides non-negative multiples of 8 elements, and
// no dimension of extent > 1 broadcast (stride 0) or rows overlapping (sn < d): every kernel reads
// the same element for a given (b, h, n) — the TMA maps and the pointer-arithmetic views alike.
cs_status check_bf16(const void* ptr, int64_t sb, int64_t sh, int64_t sn, int B, int H, int N, int d,
                     const char* name) {
  if (!ptr) return fail(CS_ERR_NULL, "%s.ptr is NULL", name);
  if (reinterpret_cast<uintptr_t>(ptr) % 16) return fail(CS_ERR_ALIGN, "%s.ptr not 16-byte aligned", name);
  if (sb < 0 || sh < 0 || sn < 0) return fail(CS_ERR_SHAPE, "%s strides must be non-negative", name);
  if (sb % 8 || sh % 8 || sn % 8)
    return fail(CS_ERR_ALIGN, "%s strides must be multiples of 8 elements (got %lld, %lld, %lld)", name,
                (long long)sb, (long long)sh, (long long)sn);
  if ((B > 1 && sb == 0) || (H > 1 && sh == 0) || (N > 1 && sn < d))
    return fail(CS_ERR_SHAPE, "%s: broadcast (stride 0) or overlapping rows (sn < d) are not supported "
                "(strides %lld, %lld, %lld for B=%d, H=%d, N=%d, d=%d)", name, (long long)sb, (long long)sh,
                (long long)sn, B, H, N, d);
  return CS_OK;
}
template <typename T>
cs_status check_t(const T& t, int B, int H, int N, int d, const char* name) {
  return check_bf16(t.ptr, t.sb, t.sh, t.sn, B, H, N, d, name);
}
cs_status check_ws(void* ws, size_t have, size_t need) {
  if (!ws) return fail(CS_ERR_WORKSPACE, "workspace is NULL (need %zu bytes)", need);
  if (reinterpret_cast<uintptr_t>(ws) % 16) return fail(CS_ERR_ALIGN, "workspace not 16-byte aligned");
  if (have < need) return fail(CS_ERR_WORKSPACE, "workspace too small: %zu < %zu bytes", have, need);
  return CS_OK;
}
#define NEED(p, name) \
  if (!(p)) return fail(CS_ERR_NULL, "%s is NULL", name)

XView view(cs_bf16_in t, int H) { return XView{static_cast<const __nv_bfloat16*>(t.ptr), t.sb, t.sh, t.sn, H}; }

// ---------------------------------------------------------------- TMA descriptors
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                  CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                  CUtensorMapFloatOOBfill);
// Driver entry points are resolved once per process (std::call_once: thread-safe); the resolved
// pointer is immutable afterwards, so the calls stay reentrant.
void* driver_entry(const char* name, std::once_flag& once, void*& slot) {
  std::call_once(once, [&] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) == cudaSuccess && q == cudaDriverEntryPointSuccess)
      slot = p;
  });
  return slot;
}
std::once_flag g_encode_once, g_attr_once;
void* g_encode_fn = nullptr;
void* g_attr_fn = nullptr;
EncodeTiledFn encode_fn() {
  return reinterpret_cast<EncodeTiledFn>(driver_entry("cuTensorMapEncodeTiled", g_encode_once, g_encode_fn));
}
// 2D bf16 map over a row-major [rows, cols] matrix, box {64, box_rows}, SWIZZLE_128B.
cs_status make_map_2d(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return fail(CS_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (no CUDA driver?)");
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(CS_ERR_CUDA, "cuTensorMapEncodeTiled (2D) failed: %d", (int)r);
  return CS_OK;
}
// 4D bf16 map over a strided [B, H, N, d] tensor, box {64, 128, 1, 1}, SWIZZLE_128B.
cs_status make_map_x(CUtensorMap* m, cs_bf16_in x, int B, int H, int N, int d) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return fail(CS_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (no CUDA driver?)");
  cuuint64_t dims[4] = {(cuuint64_t)d, (cuuint64_t)N, (cuuint64_t)H, (cuuint64_t)B};
  // real strides; only a dimension of extent 1 (never stepped over) may carry a placeholder
  // (check_bf16 rejects stride 0 on any dimension of extent > 1)
  const int64_t sn = N > 1 ? x.sn : std::max<int64_t>(x.sn, 8);
  const int64_t sh = H > 1 ? x.sh : std::max<int64_t>(x.sh, 8);
  const int64_t sb = B > 1 ? x.sb : std::max<int64_t>(x.sb, 8);
  cuuint64_t strides[3] = {(cuuint64_t)sn * 2, (cuuint64_t)sh * 2, (cuuint64_t)sb * 2};
  cuuint32_t box[4] = {64, 128, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(x.ptr), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(CS_ERR_CUDA, "cuTensorMapEncodeTiled (4D) failed: %d", (int)r);
  return CS_OK;
}

// Stage events: a plain record outside stream capture; while the stream is being captured into a
// CUDA graph, an external event-record node, so the event still times the stage in every replay.
static cudaError_t record_stage_event(void* ev, cudaStream_t st) {
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaError_t e = cudaStreamIsCapturing(st, &cap);
  if (e != cudaSuccess) return e;
  return cap == cudaStreamCaptureStatusActive
             ? cudaEventRecordWithFlags(static_cast<cudaEvent_t>(ev), st, cudaEventRecordExternal)
             : cudaEventRecord(static_cast<cudaEvent_t>(ev), st);
}

// ---------------------------------------------------------------- launch sequences
cs_status run_assign_step(int B, int H, int N, int d, cs_bf16_in x, int ka, const float* ca, int ks,
                          const float* cself, int32_t* labels, const AssignScratch& sc, cudaStream_t st) {
  const int BH = B * H;
  const int nch = chunk_n(ks), ks_pad = pad_k(ks);
  CS_CUDA(launch_anchor_prep(ca, ka, cself, ks, ks_pad, BH, d, sc.gamma, sc.wsplit, st), "anchor_prep");
  CUtensorMap tx, tw;
  CS_CHECK(make_map_x(&tx, x, B, H, N, d));
  CS_CHECK(make_map_2d(&tw, sc.wsplit, (uint64_t)BH * ks_pad, 2 * d, assign_box_rows(ks)));
  CS_CUDA(launch_assign_gemm(&tx, &tw, B, H, N, d, ks, nch, ks_pad, nullptr, labels, st), "assign_gemm");
  return CS_OK;
}

// k-means baseline half-step (NEXT-2): L(i) = argmin_j ||x_i - c_j|| through the same GEMM
cs_status run_kmeans_step(int B, int H, int N, int d, cs_bf16_in x, int ks, const float* cself, int32_t* labels,
                          const AssignScratch& sc, cudaStream_t st) {
  const int BH = B * H;
  const int nch = chunk_n(ks), ks_pad = pad_k(ks);
  CS_CUDA(launch_kmeans_prep(cself, ks, ks_pad, BH, d, sc.wsplit, sc.bias, st), "kmeans_prep");
  CUtensorMap tx, tw;
  CS_CHECK(make_map_x(&tx, x, B, H, N, d));
  CS_CHECK(make_map_2d(&tw, sc.wsplit, (uint64_t)BH * ks_pad, 2 * d, assign_box_rows(ks)));
  CS_CUDA(launch_assign_gemm(&tx, &tw, B, H, N, d, ks, nch, ks_pad, sc.bias, labels, st), "assign_gemm");
  return CS_OK;
}

cs_status run_assign(int B, int H, int N, int d, cs_bf16_in q, cs_bf16_in k, int kq, int kk, int iters,
                     uint64_t seed, int h_off, int h_tot, const int32_t* init_q, const int32_t* init_k, float* cq, float* ck,
                     int32_t* lq, int32_t* lk, int32_t* perm_q, int32_t* offs_q, int32_t* perm_k,
                     int32_t* offs_k, const AssignScratch& sc, __nv_bfloat16* qp_out,
                     __nv_bfloat16* kp_out, cudaStream_t st, bool kmeans = false) {
  const int BH = B * H;
  Nvtx range("cs.cocluster");
  const XView xq = view(q, H), xk = view(k, H);
  CS_CUDA(launch_init_sample(xq, xk, BH, N, d, kq, kk, seed, h_off, h_tot, init_q, init_k, cq, ck, st), "init_sample");
  for (int it = 0; it < iters; ++it) {
    const bool last = it == iters - 1;
    // Step A: query-aware key-side partitioning; k-means baseline: keys alone
    Nvtx ra("cs.cocluster.step_a");
    if (kmeans) CS_CHECK(run_kmeans_step(B, H, N, d, k, kk, ck, lk, sc, st));
    else CS_CHECK(run_assign_step(B, H, N, d, k, kq, cq, kk, ck, lk, sc, st));
    CS_CUDA(launch_csort(lk, BH, N, kk, perm_k, offs_k, sc.hist, st), "csort_k");
    CS_CUDA(launch_seg_mean(xk, BH, N, d, kk, perm_k, offs_k, ck, last ? kp_out : nullptr, st), "seg_mean_k");
    // Step B: key-aware query-side partitioning; k-means baseline: queries alone
    Nvtx rb("cs.cocluster.step_b");
    if (kmeans) CS_CHECK(run_kmeans_step(B, H, N, d, q, kq, cq, lq, sc, st));
    else CS_CHECK(run_assign_step(B, H, N, d, q, kk, ck, kq, cq, lq, sc, st));
    CS_CUDA(launch_csort(lq, BH, N, kq, perm_q, offs_q, sc.hist, st), "csort_q");
    CS_CUDA(launch_seg_mean(xq, BH, N, d, kq, perm_q, offs_q, cq, last ? qp_out : nullptr, st), "seg_mean_q");
  }
  return CS_OK;
}

cs_status run_attn(int B, int H, int N, int d, int kq, int kk, const int32_t* perm_q, const int32_t* offs_q,
                   const int32_t* offs_k, const int32_t* n_keep, const int32_t* n_rows, const int32_t* kept, float scale,
                   cs_bf16_out o, const AttnScratch& sc, cudaStream_t st, void* const* ev = nullptr,
                   const cs_peer_out* po = nullptr) {
  const int BH = B * H;
  Nvtx range("cs.attention");
  CS_CUDA(launch_worklist(BH, kq, offs_q, sc.item_start, st), "worklist");
  CUtensorMap tq;
  KVMaps kv;
  CS_CHECK(make_map_2d(&tq, sc.qp, (uint64_t)BH * N, d, 128));
  for (int i = 0; i < kKVBoxes; ++i) {  // box heights 8, 16, .., 128 rows (i < 5), then 1..7 rows
    const uint32_t rows = i < 5 ? 8u << i : (uint32_t)(i - 4);
    CS_CHECK(make_map_2d(&kv.k[i], sc.kp, (uint64_t)BH * N, d, rows));
    CS_CHECK(make_map_2d(&kv.v[i], sc.vp, (uint64_t)BH * N, d, rows));
  }
  if (ev) CS_CUDA(record_stage_event(ev[2], st), "event");
  CS_CUDA(launch_bsa_fwd(&tq, &kv, BH, H, N, d, kq, kk, perm_q, offs_q, offs_k, n_keep, n_rows, kept,
                         sc.item_start, worklist_upper_bound(N, kq), scale,
                         static_cast<__nv_bfloat16*>(o.ptr), o.sb, po ? po->s_head : o.sh,
                         po ? po->s_tok : o.sn, po ? static_cast<const uint64_t*>(po->ptrs) : nullptr,
                         po ? po->n_per_rank : 0, po ? po->head_base : 0, st),
          "bsa_fwd");
  if (ev) CS_CUDA(record_stage_event(ev[3], st), "event");
  return CS_OK;
}

}  // namespace

// =================================================================== exported C ABI
extern "C" {

int cs_version(void) { return 100; }

const char* cs_status_string(int s) {
  switch (s) {
    case CS_OK: return "CS_OK";
    case CS_ERR_NULL: return "CS_ERR_NULL";
    case CS_ERR_SHAPE: return "CS_ERR_SHAPE";
    case CS_ERR_ARG: return "CS_ERR_ARG";
    case CS_ERR_ALIGN: return "CS_ERR_ALIGN";
    case CS_ERR_WORKSPACE: return "CS_ERR_WORKSPACE";
    case CS_ERR_UNSUPPORTED: return "CS_ERR_UNSUPPORTED";
    case CS_ERR_CUDA: return "CS_ERR_CUDA";
  }
  return "CS_ERR_UNKNOWN";
}

const char* cs_last_error(void) { return g_err; }

size_t cs_workspace_bytes(int B, int H, int N, int d, int kq, int kk) {
  if (B <= 0 || H <= 0 || N <= 0 || kq <= 0 || kk <= 0 || (d != 64 && d != 128)) return 0;
  return need_layer(B * H, N, d, kq, kk);
}

cs_status check_heads(int H, int& h_off, int& h_tot) {
  if (h_tot == 0) {
    if (h_off != 0) return fail(CS_ERR_ARG, "head_offset must be 0 when heads_total is 0");
    h_tot = H;
  }
  if (h_off < 0 || h_off + H > h_tot)
    return fail(CS_ERR_ARG, "need 0 <= head_offset and head_offset + H <= heads_total (%d, %d, %d)", h_off, H, h_tot);
  return CS_OK;
}

static cs_status assign_entry(bool kmeans, int B, int H, int N, int d, cs_bf16_in q, cs_bf16_in k, int kq, int kk, int iters,
                         uint64_t seed, int head_offset, int heads_total, const int32_t* init_q, const int32_t* init_k, float* cq, float* ck,
                         int32_t* lq, int32_t* lk, int32_t* perm_q, int32_t* offs_q, int32_t* perm_k,
                         int32_t* offs_k, void* ws, size_t ws_bytes, void* stream) {
  g_err[0] = 0;
  CS_CHECK(check_dims(B, H, N, d));
  CS_CHECK(check_k(kq, N, "kq"));
  CS_CHECK(check_k(kk, N, "kk"));
  if (iters < 1) return fail(CS_ERR_ARG, "iters must be >= 1 (got %d)", iters);
  CS_CHECK(check_heads(H, head_offset, heads_total));
  CS_CHECK(check_t(q, B, H, N, d, "q"));
  CS_CHECK(check_t(k, B, H, N, d, "k"));
  NEED(cq, "cq"); NEED(ck, "ck"); NEED(lq, "lq"); NEED(lk, "lk");
  NEED(perm_q, "perm_q"); NEED(offs_q, "offs_q"); NEED(perm_k, "perm_k"); NEED(offs_k, "offs_k");
  const int BH = B * H;
  CS_CHECK(check_ws(ws, ws_bytes, need_assign(BH, N, d, kq, kk)));
  Carve c(ws);
  AssignScratch sc = carve_assign(c, BH, N, d, kq, kk);
  return run_assign(B, H, N, d, q, k, kq, kk, iters, seed, head_offset, heads_total, init_q, init_k, cq, ck, lq, lk, perm_q, offs_q,
                    perm_k, offs_k, sc, nullptr, nullptr, static_cast<cudaStream_t>(stream), kmeans);
}

cs_status coclust_assign(int B, int H, int N, int d, cs_bf16_in q, cs_bf16_in k, int kq, int kk, int iters,
                         uint64_t seed, int head_offset, int heads_total, const int32_t* init_q, const int32_t* init_k,
                         float* cq, float* ck, int32_t* lq, int32_t* lk, int32_t* perm_q, int32_t* offs_q,
                         int32_t* perm_k, int32_t* offs_k, void* ws, size_t ws_bytes, void* stream) {
  return assign_entry(false, B, H, N, d, q, k, kq, kk, iters, seed, head_offset, heads_total, init_q, init_k, cq, ck,
                      lq, lk, perm_q, offs_q, perm_k, offs_k, ws, ws_bytes, stream);
}

cs_status kmeans_assign(int B, int H, int N, int d, cs_bf16_in q, cs_bf16_in k, int kq, int kk, int iters,
                        uint64_t seed, int head_offset, int heads_total, const int32_t* init_q, const int32_t* init_k,
                        float* cq, float* ck, int32_t* lq, int32_t* lk, int32_t* perm_q, int32_t* offs_q,
                        int32_t* perm_k, int32_t* offs_k, void* ws, size_t ws_bytes, void* stream) {
  return assign_entry(true, B, H, N, d, q, k, kq, kk, iters, seed, head_offset, heads_total, init_q, init_k, cq, ck,
                      lq, lk, perm_q, offs_q, perm_k, offs_k, ws, ws_bytes, stream);
}

cs_status kmeans_assign_step(int B, int H, int N, int d, cs_bf16_in x, int ks, const float* c_self, int32_t* labels,
                             void* ws, size_t ws_bytes, void* stream) {
  g_err[0] = 0;
  CS_CHECK(check_dims(B, H, N, d));
  if (ks < 1 || ks > kMaxClusters) return fail(CS_ERR_ARG, "ks must be in [1, %d] (got %d)", kMaxClusters, ks);
  CS_CHECK(check_t(x, B, H, N, d, "x"));
  NEED(c_self, "c_self"); NEED(labels, "labels");
  const int BH = B * H;
  CS_CHECK(check_ws(ws, ws_bytes, need_assign(BH, N, d, ks, ks)));
  Carve c(ws);
  AssignScratch sc = carve_assign(c, BH, N, d, ks, ks);
  return run_kmeans_step(B, H, N, d, x, ks, c_self, labels, sc, static_cast<cudaStream_t>(stream));
}

cs_status coclust_assign_step(int B, int H, int N, int d, cs_bf16_in x, int ka, const float* c_anchor, int ks,
                              const float* c_self, int32_t* labels, void* ws, size_t ws_bytes, void* stream) {
  g_err[0] = 0;
  CS_CHECK(check_dims(B, H, N, d));
  if (ka < 1 || ka > kMaxClusters) return fail(CS_ERR_ARG, "ka must be in [1, %d] (got %d)", kMaxClusters, ka);
  if (ks < 1 || ks > kMaxClusters) return fail(CS_ERR_ARG, "ks must be in [1, %d] (got %d)", kMaxClusters, ks);
  CS_CHECK(check_t(x, B, H, N, d, "x"));
  NEED(c_anchor, "c_anchor"); NEED(c_self, "c_self"); NEED(labels, "labels");
  const int BH = B * H;
  CS_CHECK(check_ws(ws, ws_bytes, need_assign(BH, N, d, ka, ks)));
  Carve c(ws);
  AssignScratch sc = carve_assign(c, BH, N, d, ka, ks);
  return run_assign_step(B, H, N, d, x, ka, c_anchor, ks, c_self, labels, sc, static_cast<cudaStream_t>(stream));
}

cs_status coclust_update_centroids(int B, int H, int N, int d, cs_bf16_in x, int k, const int32_t* perm,
                                   const int32_t* offs, float* c_inout, void* x_perm, void* stream) {
  g_err[0] = 0;
  CS_CHECK(check_dims(B, H, N, d));
  CS_CHECK(check_k(k, N, "k"));
  CS_CHECK(check_t(x, B, H, N, d, "x"));
  NEED(perm, "perm"); NEED(offs, "offs"); NEED(c_inout, "c_inout");
  if (x_perm && reinterpret_cast<uintptr_t>(x_perm) % 16) return fail(CS_ERR_ALIGN, "x_perm not 16-byte aligned");
  CS_CUDA(launch_seg_mean(view(x, H), B * H, N, d, k, perm, offs, c_inout, static_cast<__nv_bfloat16*>(x_perm),
                          static_cast<cudaStream_t>(stream)),
          "seg_mean");
  return CS_OK;
}

cs_status coclust_permute(int BH, int N, int k, const int32_t* labels, int32_t* perm, int32_t* offs, void* ws,
                          size_t ws_bytes, void* stream) {
  g_err[0] = 0;
  if (BH <= 0 || N <= 0) return fail(CS_ERR_SHAPE, "BH, N must be positive");
  if (N >= (1 << 24) || (long long)BH * N >= (1LL << 31)) return fail(CS_ERR_UNSUPPORTED, "too many tokens");
  CS_CHECK(check_k(k, 1 << 30, "k"));
  NEED(labels, "labels"); NEED(perm, "perm"); NEED(offs, "offs");
  const size_t need = (size_t)BH * ((N + kSortTile - 1) / kSortTile + 1) * k * 4 + 256;
  CS_CHECK(check_ws(ws, ws_bytes, need));
  Carve c(ws);
  int32_t* hist = c.take<int32_t>((size_t)BH * ((N + kSortTile - 1) / kSortTile + 1) * k);
  CS_CUDA(launch_csort(labels, BH, N, k, perm, offs, hist, static_cast<cudaStream_t>(stream)), "csort");
  return CS_OK;
}

cs_status block_select_ex(int B, int H, int kq, int kk, int d, const float* cq, const float* ck,
                          const int32_t* offs_q, const int32_t* offs_k, const float* budget, double tau,
                          double theta, int rule, int flags, int32_t* n_keep, int32_t* n_keep_rows,
                          int32_t* kept, void* ws, size_t ws_bytes, void* stream) {
  g_err[0] = 0;
  if (B <= 0 || H <= 0) return fail(CS_ERR_SHAPE, "B, H must be positive");
  if (d != 64 && d != 128) return fail(CS_ERR_SHAPE, "d must be 64 or 128 (got %d)", d);
  CS_CHECK(check_k(kq, kMaxClusters, "kq"));
  CS_CHECK(check_k(kk, kMaxClusters, "kk"));
  if (!(tau > 0.0 && tau <= 1.0)) return fail(CS_ERR_ARG, "tau must be in (0, 1] (got %g)", tau);
  if (!(theta > 0.0 && theta < 1.0)) return fail(CS_ERR_ARG, "theta must be in (0, 1) (got %g)", theta);
  if (rule < 0 || rule > 2) return fail(CS_ERR_ARG, "unknown rule %d", rule);
  if (flags & ~(CS_SEL_PER_ROW | CS_SEL_SIZE_WEIGHTED)) return fail(CS_ERR_ARG, "unknown selection flags 0x%x", flags);
  NEED(cq, "cq"); NEED(ck, "ck"); NEED(offs_q, "offs_q"); NEED(offs_k, "offs_k"); NEED(budget, "budget");
  NEED(n_keep, "n_keep"); NEED(kept, "kept");
  if ((flags & CS_SEL_PER_ROW) && !n_keep_rows) return fail(CS_ERR_NULL, "n_keep_rows is NULL (CS_SEL_PER_ROW)");
  const int BH = B * H;
  CS_CHECK(check_ws(ws, ws_bytes, need_select(BH, kq, kk)));
  Carve c(ws);
  SelectScratch sc = carve_select(c, BH, kq, kk);
  CS_CUDA(launch_block_select(BH, H, kq, kk, d, cq, ck, offs_q, offs_k, budget, tau, theta, rule, flags, n_keep,
                              n_keep_rows, kept, sc.order, sc.cnt, sc.abar, static_cast<cudaStream_t>(stream)),
          "block_select");
  return CS_OK;
}

cs_status block_select(int B, int H, int kq, int kk, int d, const float* cq, const float* ck,
                       const int32_t* offs_q, const int32_t* offs_k, const float* budget, double tau,
                       double theta, int rule, int32_t* n_keep, int32_t* kept, void* ws, size_t ws_bytes,
                       void* stream) {
  return block_select_ex(B, H, kq, kk, d, cq, ck, offs_q, offs_k, budget, tau, theta, rule, 0, n_keep, nullptr,
                         kept, ws, ws_bytes, stream);
}

cs_status block_sparse_attn_ex(int B, int H, int N, int d, cs_bf16_in q, cs_bf16_in k, cs_bf16_in v, int kq,
                               int kk, const int32_t* perm_q, const int32_t* offs_q, const int32_t* perm_k,
                               const int32_t* offs_k, const int32_t* n_keep, const int32_t* n_keep_rows,
                               const int32_t* kept, float scale, cs_bf16_out o, void* ws, size_t ws_bytes,
                               void* stream) {
  g_err[0] = 0;
  CS_CHECK(check_dims(B, H, N, d));
  CS_CHECK(check_k(kq, N, "kq"));
  CS_CHECK(check_k(kk, N, "kk"));
  CS_CHECK(check_t(q, B, H, N, d, "q"));
  CS_CHECK(check_t(k, B, H, N, d, "k"));
  CS_CHECK(check_t(v, B, H, N, d, "v"));
  CS_CHECK(check_t(o, B, H, N, d, "o"));
  if (!(scale > 0.f)) return fail(CS_ERR_ARG, "scale must be > 0 (got %g)", (double)scale);
  NEED(perm_q, "perm_q"); NEED(offs_q, "offs_q"); NEED(perm_k, "perm_k"); NEED(offs_k, "offs_k");
  NEED(n_keep, "n_keep"); NEED(kept, "kept");
  const int BH = B * H;
  CS_CHECK(check_ws(ws, ws_bytes, need_attn(BH, N, d, kq)));
  Carve c(ws);
  AttnScratch sc = carve_attn(c, BH, N, d, kq);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  CS_CUDA(launch_permute_rows(view(q, H), BH, N, d, perm_q, sc.qp, st), "permute_q");
  CS_CUDA(launch_permute_rows(view(k, H), BH, N, d, perm_k, sc.kp, st), "permute_k");
  CS_CUDA(launch_permute_rows(view(v, H), BH, N, d, perm_k, sc.vp, st), "permute_v");
  return run_attn(B, H, N, d, kq, kk, perm_q, offs_q, offs_k, n_keep, n_keep_rows, kept, scale, o, sc, st);
}

cs_status block_sparse_attn(int B, int H, int N, int d, cs_bf16_in q, cs_bf16_in k, cs_bf16_in v, int kq, int kk,
                            const int32_t* perm_q, const int32_t* offs_q, const int32_t* perm_k,
                            const int32_t* offs_k, const int32_t* n_keep, const int32_t* kept, float scale,
                            cs_bf16_out o, void* ws, size_t ws_bytes, void* stream) {
  return block_sparse_attn_ex(B, H, N, d, q, k, v, kq, kk, perm_q, offs_q, perm_k, offs_k, n_keep, nullptr, kept,
                              scale, o, ws, ws_bytes, stream);
}

}  // extern "C"

namespace {
cs_status check_layer_args(int B, int H, int N, int d, cs_bf16_in q, cs_bf16_in k, cs_bf16_in v, int kq, int kk,
                           int iters, int& head_offset, int& heads_total, const float* budget, double tau,
                           double theta, int rule, int sel_flags, float scale, cs_bf16_out o) {
  CS_CHECK(check_dims(B, H, N, d));
  CS_CHECK(check_k(kq, N, "kq"));
  CS_CHECK(check_k(kk, N, "kk"));
  if (iters < 1) return fail(CS_ERR_ARG, "iters must be >= 1 (got %d)", iters);
  if (!(tau > 0.0 && tau <= 1.0)) return fail(CS_ERR_ARG, "tau must be in (0, 1] (got %g)", tau);
  if (!(theta > 0.0 && theta < 1.0)) return fail(CS_ERR_ARG, "theta must be in (0, 1) (got %g)", theta);
  if (rule < 0 || rule > 2) return fail(CS_ERR_ARG, "unknown rule %d", rule);
  if (sel_flags & ~(CS_SEL_PER_ROW | CS_SEL_SIZE_WEIGHTED | CS_CLUSTER_KMEANS))
    return fail(CS_ERR_ARG, "unknown flags 0x%x", sel_flags);
  if (!(scale > 0.f)) return fail(CS_ERR_ARG, "scale must be > 0 (got %g)", (double)scale);
  CS_CHECK(check_heads(H, head_offset, heads_total));
  CS_CHECK(check_t(q, B, H, N, d, "q"));
  CS_CHECK(check_t(k, B, H, N, d, "k"));
  CS_CHECK(check_t(v, B, H, N, d, "v"));
  CS_CHECK(check_t(o, B, H, N, d, "o"));
  NEED(budget, "budget");
  return CS_OK;
}

// The whole layer on device.  recompute: co-cluster + select into `s`; otherwise reuse `s`.
cs_status run_layer(int B, int H, int N, int d, cs_bf16_in q, cs_bf16_in k, cs_bf16_in v, int kq, int kk,
                    int iters, uint64_t seed, int head_offset, int heads_total, const float* budget, double tau,
                    double theta, int rule, int sel_flags, float scale, cs_bf16_out o, const LayerState& s, bool recompute,
                    Carve& c, cudaStream_t st, void* const* ev, const cs_peer_out* po = nullptr,
                    void* v_ready = nullptr) {
  const int BH = B * H;
  AttnScratch at = carve_attn(c, BH, N, d, kq);
  AssignScratch as = carve_assign(c, BH, N, d, kq, kk);
  SelectScratch se = carve_select(c, BH, kq, kk);
  if (recompute) {
    CS_CHECK(run_assign(B, H, N, d, q, k, kq, kk, iters, seed, head_offset, heads_total, nullptr, nullptr, s.cq,
                        s.ck, s.lq, s.lk, s.perm_q, s.offs_q, s.perm_k, s.offs_k, as, at.qp, at.kp, st,
                        (sel_flags & CS_CLUSTER_KMEANS) != 0));
    if (ev) CS_CUDA(record_stage_event(ev[0], st), "event");
    Nvtx rs("cs.select");
    CS_CUDA(launch_block_select(BH, H, kq, kk, d, s.cq, s.ck, s.offs_q, s.offs_k, budget, tau, theta, rule,
                                sel_flags & (CS_SEL_PER_ROW | CS_SEL_SIZE_WEIGHTED), s.n_keep, s.n_rows, s.kept,
                                se.order, se.cnt, se.abar, st),
            "block_select");
    if (ev) CS_CUDA(record_stage_event(ev[1], st), "event");
  } else {
    // clustering reuse across denoising steps: only the permuted copies are new
    if (ev) CS_CUDA(record_stage_event(ev[0], st), "event");
    CS_CUDA(launch_permute_rows(view(q, H), BH, N, d, s.perm_q, at.qp, st), "permute_q");
    CS_CUDA(launch_permute_rows(view(k, H), BH, N, d, s.perm_k, at.kp, st), "permute_k");
    if (ev) CS_CUDA(record_stage_event(ev[1], st), "event");
  }
  // V is first read here: a caller still delivering it on another stream (the Ulysses in-bound
  // all-to-all of V overlapping the co-clustering, which reads only Q and K) passes its event
  if (v_ready) CS_CUDA(cudaStreamWaitEvent(st, static_cast<cudaEvent_t>(v_ready), 0), "wait v_ready");
  CS_CUDA(launch_permute_rows(view(v, H), BH, N, d, s.perm_k, at.vp, st), "permute_v");
  return run_attn(B, H, N, d, kq, kk, s.perm_q, s.offs_q, s.offs_k, s.n_keep, s.n_rows, s.kept, scale, o, at, st,
                  ev, po);
}
}  // namespace

extern "C" {

cs_status coclust_sparse_attention_ex(int B, int H, int N, int d, cs_bf16_in q, cs_bf16_in k, cs_bf16_in v,
                                      int kq, int kk, int iters, uint64_t seed, int head_offset, int heads_total,
                                      const float* budget, double tau, double theta, int rule, int sel_flags,
                                      float scale, cs_bf16_out o, void* ws, size_t ws_bytes, void* stream,
                                      void* const* stage_events) {
  g_err[0] = 0;
  CS_CHECK(check_layer_args(B, H, N, d, q, k, v, kq, kk, iters, head_offset, heads_total, budget, tau, theta,
                            rule, sel_flags, scale, o));
  const int BH = B * H;
  CS_CHECK(check_ws(ws, ws_bytes, need_layer(BH, N, d, kq, kk)));
  Carve c(ws);
  LayerState s = carve_state(c, BH, N, d, kq, kk);
  return run_layer(B, H, N, d, q, k, v, kq, kk, iters, seed, head_offset, heads_total, budget, tau, theta, rule,
                   sel_flags, scale, o, s, true, c, static_cast<cudaStream_t>(stream), stage_events);
}

cs_status coclust_sparse_attention(int B, int H, int N, int d, cs_bf16_in q, cs_bf16_in k, cs_bf16_in v, int kq,
                                   int kk, int iters, uint64_t seed, int head_offset, int heads_total,
                                   const float* budget, double tau, double theta,
                                   int rule, float scale, cs_bf16_out o, void* ws, size_t ws_bytes, void* stream,
                                   void* const* stage_events) {
  return coclust_sparse_attention_ex(B, H, N, d, q, k, v, kq, kk, iters, seed, head_offset, heads_total, budget,
                                     tau, theta, rule, 0, scale, o, ws, ws_bytes, stream, stage_events);
}

cs_status coclust_sparse_attention_cached(int B, int H, int N, int d, cs_bf16_in q, cs_bf16_in k, cs_bf16_in v,
                                          int kq, int kk, int iters, uint64_t seed, int head_offset,
                                          int heads_total, const float* budget, double tau, double theta, int rule,
                                          int sel_flags, float scale, cs_bf16_out o, const cs_layer_state* state,
                                          int recompute,
                                          void* ws, size_t ws_bytes, void* stream, void* const* stage_events) {
  g_err[0] = 0;
  CS_CHECK(check_layer_args(B, H, N, d, q, k, v, kq, kk, iters, head_offset, heads_total, budget, tau, theta,
                            rule, sel_flags, scale, o));
  NEED(state, "state");
  if ((sel_flags & CS_SEL_PER_ROW) && !state->n_keep_rows)
    return fail(CS_ERR_NULL, "state->n_keep_rows is NULL (CS_SEL_PER_ROW)");
  NEED(state->cq, "state->cq"); NEED(state->ck, "state->ck"); NEED(state->lq, "state->lq");
  NEED(state->lk, "state->lk"); NEED(state->perm_q, "state->perm_q"); NEED(state->offs_q, "state->offs_q");
  NEED(state->perm_k, "state->perm_k"); NEED(state->offs_k, "state->offs_k");
  NEED(state->n_keep, "state->n_keep"); NEED(state->kept, "state->kept");
  const int BH = B * H;
  Carve dry(nullptr);
  carve_attn(dry, BH, N, d, kq);
  carve_assign(dry, BH, N, d, kq, kk);
  carve_select(dry, BH, kq, kk);
  CS_CHECK(check_ws(ws, ws_bytes, dry.off + 256));
  LayerState s{state->cq, state->ck, state->lq, state->lk, state->perm_q, state->perm_k, state->offs_q,
               state->offs_k, state->n_keep, state->kept, state->n_keep_rows};
  Carve c(ws);
  return run_layer(B, H, N, d, q, k, v, kq, kk, iters, seed, head_offset, heads_total, budget, tau, theta, rule,
                   sel_flags, scale, o, s, recompute != 0, c, static_cast<cudaStream_t>(stream), stage_events);
}

size_t cs_density_workspace_bytes(int B, int H, int N) {
  if (B <= 0 || H <= 0 || N <= 0) return 0;
  Carve c(nullptr);
  const size_t rows = (size_t)B * H * N;
  c.take<float>(6 * rows);
  c.take<int32_t>(rows);
  return c.off + 256;
}

cs_status attention_density(int B, int H, int N, int d, cs_bf16_in q, cs_bf16_in k, double tau, float scale,
                            int passes, int32_t* counts, double* density, void* ws, size_t ws_bytes, void* stream) {
  g_err[0] = 0;
  CS_CHECK(check_dims(B, H, N, d));
  CS_CHECK(check_t(q, B, H, N, d, "q"));
  CS_CHECK(check_t(k, B, H, N, d, "k"));
  if (!(tau > 0.0 && tau <= 1.0)) return fail(CS_ERR_ARG, "tau must be in (0, 1] (got %g)", tau);
  if (!(scale > 0.f)) return fail(CS_ERR_ARG, "scale must be > 0 (got %g)", (double)scale);
  if (passes == 0) passes = 4;
  if (passes < 1 || passes > 5) return fail(CS_ERR_ARG, "passes must be in [1, 5] (got %d)", passes);
  NEED(density, "density");
  CS_CHECK(check_ws(ws, ws_bytes, cs_density_workspace_bytes(B, H, N)));
  Carve c(ws);
  const size_t rows = (size_t)B * H * N;
  float* st6 = c.take<float>(6 * rows);
  int32_t* cnt = c.take<int32_t>(rows);
  CUtensorMap tq, tk;
  CS_CHECK(make_map_x(&tq, q, B, H, N, d));
  CS_CHECK(make_map_x(&tk, k, B, H, N, d));
  CS_CUDA(launch_attention_density(&tq, &tk, B, H, N, d, scale, tau, passes, st6, rows, counts ? counts : cnt,
                                   density, static_cast<cudaStream_t>(stream)),
          "attention_density");
  return CS_OK;
}

cs_status coclust_sparse_attention_peer(int H, int N, int d, cs_bf16_in q, cs_bf16_in k, cs_bf16_in v, int kq,
                                        int kk, int iters, uint64_t seed, int head_offset, int heads_total,
                                        const float* budget, double tau, double theta, int rule, int flags,
                                        float scale, const cs_peer_out* o, void* ws, size_t ws_bytes, void* stream,
                                        void* const* stage_events) {
  g_err[0] = 0;
  NEED(o, "o");
  NEED(o->ptrs, "o->ptrs");
  if (o->P < 1 || o->n_per_rank < 1 || (long long)o->P * o->n_per_rank != N)
    return fail(CS_ERR_SHAPE, "peer output: P * n_per_rank must equal N (%d * %d vs %d)", o->P, o->n_per_rank, N);
  if (o->head_base < 0 || o->s_tok <= 0 || o->s_head <= 0 || o->s_tok % 8 || o->s_head % 8)
    return fail(CS_ERR_ALIGN, "peer output: strides must be positive multiples of 8 elements");
  cs_bf16_out dummy{const_cast<void*>(o->ptrs), 0, o->s_head, o->s_tok};  // validated like an output, never stored to
  CS_CHECK(check_layer_args(1, H, N, d, q, k, v, kq, kk, iters, head_offset, heads_total, budget, tau, theta,
                            rule, flags, scale, dummy));
  CS_CHECK(check_ws(ws, ws_bytes, need_layer(H, N, d, kq, kk)));
  Carve c(ws);
  LayerState s = carve_state(c, H, N, d, kq, kk);
  return run_layer(1, H, N, d, q, k, v, kq, kk, iters, seed, head_offset, heads_total, budget, tau, theta, rule,
                   flags, scale, dummy, s, true, c, static_cast<cudaStream_t>(stream), stage_events, o);
}

cs_status coclust_sparse_attention_ulysses(int H, int N, int d, cs_bf16_in q, cs_bf16_in k, cs_bf16_in v, int kq,
                                           int kk, int iters, uint64_t seed, int head_offset, int heads_total,
                                           const float* budget, double tau, double theta, int rule, int flags,
                                           float scale, cs_bf16_out o, const cs_peer_out* peer, void* v_ready,
                                           void* ws, size_t ws_bytes, void* stream, void* const* stage_events) {
  g_err[0] = 0;
  cs_bf16_out out = o;
  if (peer) {
    NEED(peer->ptrs, "peer->ptrs");
    if (peer->P < 1 || peer->n_per_rank < 1 || (long long)peer->P * peer->n_per_rank != N)
      return fail(CS_ERR_SHAPE, "peer output: P * n_per_rank must equal N (%d * %d vs %d)", peer->P,
                  peer->n_per_rank, N);
    if (peer->head_base < 0 || peer->s_tok <= 0 || peer->s_head <= 0 || peer->s_tok % 8 || peer->s_head % 8)
      return fail(CS_ERR_ALIGN, "peer output: strides must be positive multiples of 8 elements");
    out = cs_bf16_out{const_cast<void*>(peer->ptrs), 0, peer->s_head, peer->s_tok};  // validated, never stored to
  }
  CS_CHECK(check_layer_args(1, H, N, d, q, k, v, kq, kk, iters, head_offset, heads_total, budget, tau, theta,
                            rule, flags, scale, out));
  CS_CHECK(check_ws(ws, ws_bytes, need_layer(H, N, d, kq, kk)));
  Carve c(ws);
  LayerState s = carve_state(c, H, N, d, kq, kk);
  return run_layer(1, H, N, d, q, k, v, kq, kk, iters, seed, head_offset, heads_total, budget, tau, theta, rule,
                   flags, scale, out, s, true, c, static_cast<cudaStream_t>(stream), stage_events, peer, v_ready);
}

cs_status cs_ulysses_pack_group(int Nl, int P, int Hl, int Hg, int g, int d, int T, const void* const* srcs,
                                void* dst, void* stream) {
  g_err[0] = 0;
  if (Nl <= 0 || P <= 0 || Hl <= 0 || (d != 64 && d != 128)) return fail(CS_ERR_SHAPE, "Nl, P, Hl > 0, d in {64, 128}");
  if (Hg <= 0 || Hl % Hg || g < 0 || g >= Hl / Hg)
    return fail(CS_ERR_ARG, "need Hg > 0 dividing Hl and 0 <= g < Hl / Hg (Hl %d, Hg %d, g %d)", Hl, Hg, g);
  if (T < 1 || T > 4) return fail(CS_ERR_ARG, "T must be in [1, 4] (got %d)", T);
  NEED(srcs, "srcs"); NEED(dst, "dst");
  UlyssesSrcs u{};
  for (int t = 0; t < T; ++t) {
    NEED(srcs[t], "srcs[t]");
    if (reinterpret_cast<uintptr_t>(srcs[t]) % 16) return fail(CS_ERR_ALIGN, "srcs[%d] not 16-byte aligned", t);
    u.p[t] = static_cast<const uint4*>(srcs[t]);
  }
  if (reinterpret_cast<uintptr_t>(dst) % 16) return fail(CS_ERR_ALIGN, "dst not 16-byte aligned");
  CS_CUDA(launch_ulysses_pack(Nl, P, T, (size_t)Hg * d * 2, (size_t)Hl * d * 2, (size_t)g * Hg * d * 2, u, dst,
                              static_cast<cudaStream_t>(stream)),
          "ulysses_pack");
  return CS_OK;
}

cs_status cs_ulysses_pack(int Nl, int P, int Hl, int d, int T, const void* const* srcs, void* dst, void* stream) {
  return cs_ulysses_pack_group(Nl, P, Hl, Hl, 0, d, T, srcs, dst, stream);
}

cs_status cs_peer_barrier(int P, int rank, const void* peer_flags, int epoch, void* stream) {
  g_err[0] = 0;
  if (P < 1 || P > 32 || rank < 0 || rank >= P) return fail(CS_ERR_ARG, "need 1 <= P <= 32, 0 <= rank < P");
  if (epoch < 1) return fail(CS_ERR_ARG, "epoch must be >= 1 (flags start at 0)");
  NEED(peer_flags, "peer_flags");
  CS_CUDA(launch_peer_barrier(P, rank, static_cast<const uint64_t*>(peer_flags), epoch,
                              static_cast<cudaStream_t>(stream)),
          "peer_barrier");
  return CS_OK;
}

typedef CUresult (*PtrAttrFn)(void*, CUpointer_attribute, CUdeviceptr);

cs_status cs_ipc_handle(const void* dev_ptr, void* handle_out, size_t* offset_out) {
  g_err[0] = 0;
  NEED(dev_ptr, "dev_ptr"); NEED(handle_out, "handle_out"); NEED(offset_out, "offset_out");
  PtrAttrFn attr = reinterpret_cast<PtrAttrFn>(driver_entry("cuPointerGetAttribute", g_attr_once, g_attr_fn));
  if (!attr) return fail(CS_ERR_CUDA, "cuPointerGetAttribute unavailable");
  CUdeviceptr base = 0;
  if (attr(&base, CU_POINTER_ATTRIBUTE_RANGE_START_ADDR, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS)
    return fail(CS_ERR_CUDA, "cuPointerGetAttribute(RANGE_START_ADDR) failed");
  cudaIpcMemHandle_t h;
  CS_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)), "cudaIpcGetMemHandle");
  memcpy(handle_out, &h, sizeof(h));
  *offset_out = reinterpret_cast<uintptr_t>(dev_ptr) - static_cast<uintptr_t>(base);
  return CS_OK;
}

cs_status cs_ipc_open(const void* handle, size_t offset, void** dev_ptr_out) {
  g_err[0] = 0;
  NEED(handle, "handle"); NEED(dev_ptr_out, "dev_ptr_out");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  void* base = nullptr;
  CS_CUDA(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
  *dev_ptr_out = static_cast<uint8_t*>(base) + offset;
  return CS_OK;
}

cs_status cs_ipc_close(void* dev_ptr, size_t offset) {
  g_err[0] = 0;
  NEED(dev_ptr, "dev_ptr");
  CS_CUDA(cudaIpcCloseMemHandle(static_cast<uint8_t*>(dev_ptr) - offset), "cudaIpcCloseMemHandle");
  return CS_OK;
}

cs_status cs_block_transpose(int A, int B, size_t row_bytes, const void* src, void* dst, void* stream) {
  g_err[0] = 0;
  if (A <= 0 || B <= 0 || row_bytes == 0) return fail(CS_ERR_SHAPE, "A, B, row_bytes must be positive");
  if (row_bytes % 16) return fail(CS_ERR_ALIGN, "row_bytes must be a multiple of 16 (got %zu)", row_bytes);
  NEED(src, "src"); NEED(dst, "dst");
  if (reinterpret_cast<uintptr_t>(src) % 16 || reinterpret_cast<uintptr_t>(dst) % 16)
    return fail(CS_ERR_ALIGN, "src/dst must be 16-byte aligned");
  CS_CUDA(launch_block_transpose(A, B, row_bytes, src, dst, static_cast<cudaStream_t>(stream)), "block_transpose");
  return CS_OK;
}

}  // extern "C"
