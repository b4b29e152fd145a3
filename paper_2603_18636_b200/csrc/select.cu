// select.cu — top block-pair selection and the attention work list.
//   k_select_rows : per (bh, query block a): Abar_a = C_q[a] C_k^T (fp64, empty key blocks -> -inf),
//                   order = key blocks by (Abar desc, index asc) (bitonic sort of 32-bit keys,
//                   exact fix-up of truncated-key collisions),
//                   c_a = min{m : cumsum of softmax(Abar_a / sqrt(d)) over that order >= tau-1e-12}
//   k_select_count: per bh: n_rec = ceil(sum c_a / Kq'), rule (R8, R10) -> n_keep
//   k_select_emit : kept[a] = the first n_keep of order[a], ascending
//   k_worklist    : per bh, exclusive scan of ceil(ceil(|Q_a|/128)/2) -> attention work items
#include <float.h>

#include "kernels.cuh"

namespace cs {

// Abar = C_q C_k^T in fp64.  grid (ceil(kk/64), ceil(kq/64), BH), block 256, dyn smem
// 2 x 64 x (64+1) doubles: a 64 x 64 output tile; thread (ta, tj) = (t / 16, t % 16) owns the
// outputs (a0 + ta + 16 i, j0 + tj + 16 jj), i, jj < 4, each a dot product of length D in a fixed
// (sequential) order, the D columns staged through SMEM in chunks of 64.  Rows padded to 65
// doubles: the 16 lanes of a half-warp hit 16 distinct bank pairs; 8 SMEM wavefronts per 16 DFMA.
template <int D>
__global__ void __launch_bounds__(256) k_abar(int kq, int kk, const float* __restrict__ cq,
                                              const float* __restrict__ ck, double* __restrict__ abar) {
  constexpr int TA = 64, TJ = 64, EC = 64, LD = EC + 1;
  extern __shared__ double sm_ab[];
  double* sq = sm_ab;             // [TA][LD]
  double* sk = sm_ab + TA * LD;   // [TJ][LD]
  const int bh = blockIdx.z, a0 = blockIdx.y * TA, j0 = blockIdx.x * TJ, t = threadIdx.x;
  const int ta = t >> 4, tj = t & 15;
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) acc[i][jj] = 0.0;
  for (int e0 = 0; e0 < D; e0 += EC) {
    if (e0) __syncthreads();
    for (int i = t; i < TA * EC / 4; i += 256) {
      const int r = i / (EC / 4), c = (i % (EC / 4)) * 4;
      const float4 v = (a0 + r < kq) ? *reinterpret_cast<const float4*>(cq + ((size_t)bh * kq + a0 + r) * D + e0 + c)
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
      double* d = sq + r * LD + c;
      d[0] = v.x; d[1] = v.y; d[2] = v.z; d[3] = v.w;
    }
    for (int i = t; i < TJ * EC / 4; i += 256) {
      const int r = i / (EC / 4), c = (i % (EC / 4)) * 4;
      const float4 v = (j0 + r < kk) ? *reinterpret_cast<const float4*>(ck + ((size_t)bh * kk + j0 + r) * D + e0 + c)
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
      double* d = sk + r * LD + c;
      d[0] = v.x; d[1] = v.y; d[2] = v.z; d[3] = v.w;
    }
    __syncthreads();
#pragma unroll 4
    for (int e = 0; e < EC; ++e) {
      double qv[4], kv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) qv[i] = sq[(ta + 16 * i) * LD + e];
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) kv[jj] = sk[(tj + 16 * jj) * LD + e];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) acc[i][jj] = fma(qv[i], kv[jj], acc[i][jj]);
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int a = a0 + ta + 16 * i;
    if (a >= kq) continue;
    double* row = abar + ((size_t)bh * kq + a) * kk;
#pragma unroll
    for (int jj = 0; jj < 4; ++jj)
      if (j0 + tj + 16 * jj < kk) row[j0 + tj + 16 * jj] = acc[i][jj];
  }
}

// Order-preserving 32-bit sort key of (value desc, index asc): the value rounded to float (round to
// nearest is monotone non-decreasing; -0 folded into +0 so that the two zeros, equal as doubles,
// tie), its sign-flipped bits truncated to 22 bits (still monotone), then 1023 - j in the low 10
// bits (K_k <= 1024), so that a larger key comes first and equal truncated values fall back to the
// lower index.  Distinct doubles whose truncated keys collide are put back into exact order after
// the sort (fixup_runs); all other pairs are already ordered exactly.
static_assert(kMaxClusters <= 1024, "sort_key packs the key-block index into 10 bits");
__device__ __forceinline__ uint32_t sort_key(double v, int j) {
  uint32_t u = __float_as_uint(__double2float_rn(v));
  if ((u << 1) == 0u) u = 0u;  // -0 -> +0 (bitwise, so no compiler flag can fold it away)
  u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  return ((u >> 10) << 10) | (uint32_t)(1023 - j);
}
__device__ __forceinline__ int key_index(uint32_t k) { return 1023 - (int)(k & 1023u); }

// Block-wide bitonic sort (descending) of P2 = 256 E distinct 32-bit keys.  Thread t holds the E
// consecutive entries t E .. t E + E - 1 in registers: strides < E are resolved inside the thread,
// strides < 32 E with warp shuffles, and only the strides >= 32 E go through shared memory.
template <int E>
__device__ void bitonic_sort_keys(uint32_t (&k)[E], int P2, uint32_t* skey) {
  const int t = threadIdx.x;
  for (int size = 2; size <= P2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      if (stride < E) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          if (e & stride) continue;
          const int e2 = e | stride;
          const bool up = ((t * E + e) & size) == 0;
          const uint32_t a = k[e], b = k[e2];
          const bool sw = up ? (b > a) : (a > b);
          k[e] = sw ? b : a;
          k[e2] = sw ? a : b;
        }
      } else {
        uint32_t ko[E];
        if (stride < 32 * E) {
#pragma unroll
          for (int e = 0; e < E; ++e) ko[e] = __shfl_xor_sync(0xffffffffu, k[e], stride / E);
        } else {
#pragma unroll
          for (int e = 0; e < E; ++e) skey[t * E + e] = k[e];
          __syncthreads();
#pragma unroll
          for (int e = 0; e < E; ++e) ko[e] = skey[(t * E + e) ^ stride];
          __syncthreads();
        }
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int i = t * E + e;
          const bool lower = (i & stride) == 0, up = (i & size) == 0;
          // keep the larger key where (lower == up), the smaller one elsewhere
          k[e] = (lower == up) ? max(k[e], ko[e]) : min(k[e], ko[e]);
        }
      }
    }
  }
#pragma unroll
  for (int e = 0; e < E; ++e) skey[t * E + e] = k[e];
  __syncthreads();
}

// grid (kq, BH), block 256, dyn smem: 2 P2 doubles + P2 uint32; P2 = 256 E
template <int E>
__global__ void __launch_bounds__(256) k_select_rows(int kq, int kk, int d, const double* __restrict__ abar,
                                                     const int32_t* __restrict__ offs_q,
                                                     const int32_t* __restrict__ offs_k, double tau,
                                                     int weighted, int need_cnt, int32_t* __restrict__ order,
                                                     int32_t* __restrict__ cnt) {
  extern __shared__ double sh_d[];
  __shared__ double wred[8];
  __shared__ int first_hit;
  constexpr int P2 = 256 * E;
  double* sval = sh_d;                 // [P2] values in sorted order
  double* vbyj = sh_d + P2;            // [P2] values by key-block index
  uint32_t* skey = reinterpret_cast<uint32_t*>(vbyj + P2);  // [P2] sorted keys
  const int a = blockIdx.x, bh = blockIdx.y, t = threadIdx.x;
  const int32_t* ok = offs_k + (size_t)bh * (kk + 1);
  const int32_t* oq = offs_q + (size_t)bh * (kq + 1);
  const double* arow = abar + ((size_t)bh * kq + a) * kk;
  // sort: (value desc, index asc); empty key blocks and padding are -inf.  The value is the raw
  // Abar (R7), or with CS_SEL_SIZE_WEIGHTED the importance Abar / sqrt(d) + log|K_c| (R9c).
  const double sdiv = weighted ? 1.0 : sqrt((double)d);  // softmax argument = value / sdiv
  {
    uint32_t key[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int j = t * E + e;
      const int sz = j < kk ? ok[j + 1] - ok[j] : 0;
      const double v = sz > 0 ? (weighted ? arow[j] / sqrt((double)d) + log((double)sz) : arow[j]) : -INFINITY;
      vbyj[j] = v;
      key[e] = sort_key(v, j);
    }
    bitonic_sort_keys<E>(key, P2, skey);
  }
#pragma unroll
  for (int e = 0; e < E; ++e) sval[t * E + e] = vbyj[key_index(skey[t * E + e])];
  __syncthreads();
  // fixup_runs: a run of equal truncated keys holding distinct values is re-ordered exactly by
  // (value desc, index asc) by the thread owning its first entry (insertion sort; runs are short
  // and rare, and a run of equal values is already in index order).  The runs are found before any
  // thread reorders one (reads and writes of the arrays in separate phases).
  int run_b[E], run_e[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = t * E + e;
    const uint32_t hk = skey[i] >> 10;
    run_b[e] = run_e[e] = i;
    if (i + 1 >= P2 || (skey[i + 1] >> 10) != hk || (i > 0 && (skey[i - 1] >> 10) == hk)) continue;
    int r = i + 1;
    while (r < P2 && (skey[r] >> 10) == hk) ++r;
    run_e[e] = r;
  }
  __syncthreads();
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = run_b[e], r = run_e[e];
    for (int x = i + 1; x < r; ++x) {
      const uint32_t kx = skey[x];
      const double vx = sval[x];
      int y = x - 1;
      while (y >= i && (sval[y] < vx || (sval[y] == vx && key_index(skey[y]) > key_index(kx)))) {
        skey[y + 1] = skey[y];
        sval[y + 1] = sval[y];
        --y;
      }
      skey[y + 1] = kx;
      sval[y + 1] = vx;
    }
  }
  __syncthreads();
  int32_t* ord = order + ((size_t)bh * kq + a) * kk;
  for (int j = t; j < kk; j += 256) ord[j] = key_index(skey[j]);
  // the FIXED rule keeps n_b blocks whatever the recall counts are: c_a is not computed
  if (!need_cnt) {
    if (t == 0) cnt[(size_t)bh * kq + a] = 0;
    return;
  }
  // number of nonempty key blocks
  int ne = 0;
  for (int j = t; j < kk; j += 256) ne += (ok[j + 1] - ok[j] > 0) ? 1 : 0;
  ne = warp_sum(ne);
  __shared__ int sne[8];
  if ((t & 31) == 0) sne[t >> 5] = ne;
  __syncthreads();
  int kne = 0;
  for (int w = 0; w < 8; ++w) kne += sne[w];
  const bool q_nonempty = oq[a + 1] - oq[a] > 0;
  if (!q_nonempty || kne == 0) {
    if (t == 0) cnt[(size_t)bh * kq + a] = 0;
    return;
  }
  // softmax over the kne nonempty entries (sorted prefix), then the cumulative mass
  const double sd = sdiv;
  const double mz = sval[0] / sd;
  // each thread owns 4 consecutive sorted entries (P2 <= 1024)
  constexpr int per = E;
  double e_loc[E];
  double s_loc = 0.0;
  for (int u = 0; u < per; ++u) {
    const int i = t * per + u;
    e_loc[u] = (i < kne) ? exp(sval[i] / sd - mz) : 0.0;
    s_loc += e_loc[u];
  }
  // block sum (fixed tree order)
  double tot = s_loc;
  for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
  if ((t & 31) == 0) wred[t >> 5] = tot;
  __syncthreads();
  double total = 0.0;
  for (int w = 0; w < 8; ++w) total += wred[w];
  __syncthreads();
  // exclusive scan of the per-thread sums of p
  double p_loc = 0.0;
  for (int u = 0; u < per; ++u) { e_loc[u] /= total; p_loc += e_loc[u]; }
  double x = p_loc;
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, x, o);
    if ((t & 31) >= o) x += y;
  }
  if ((t & 31) == 31) wred[t >> 5] = x;
  if (t == 0) first_hit = kne;
  __syncthreads();
  double base = 0.0;
  for (int w = 0; w < (t >> 5); ++w) base += wred[w];
  double cs_ = base + x - p_loc;
  const double thr = tau - 1e-12;
  for (int u = 0; u < per; ++u) {
    const int i = t * per + u;
    cs_ += e_loc[u];
    if (i < kne && cs_ >= thr) { atomicMin(&first_hit, i + 1); break; }
  }
  __syncthreads();
  if (t == 0) cnt[(size_t)bh * kq + a] = first_hit;
}

__device__ __forceinline__ int n_from_ratio(double r, int kk) {
  int n = (int)ceil(r * (double)kk - 1e-3);
  return min(max(n, 1), kk);
}

// the rho rule (R8, R10) for a recall count n_rec, clamped to [1, K_k']
__device__ __forceinline__ int rule_n(int n_rec, double b, double theta, int rule, int kk, int nk) {
  const int n_b = n_from_ratio(b, kk);
  int n;
  if (rule == 0) n = (1.0 - b) > theta ? min(n_rec, n_b) : max(n_rec, n_b);
  else if (rule == 1) n = b > theta ? min(n_rec, n_b) : max(n_rec, n_b);
  else n = n_b;
  return min(max(n, 1), max(nk, 1));
}

// grid BH, block 1024.  n_keep[bh] = rule(n_rec) (R11).  n_rows (optional) gets the per-row
// counts: with per_row (CS_SEL_PER_ROW, R11b) rule(c_a) for nonempty query blocks and the shared
// n for empty ones; without it the shared n everywhere.
__global__ void __launch_bounds__(1024) k_select_count(int H, int kq, int kk,
                                                       const int32_t* __restrict__ offs_q,
                                                       const int32_t* __restrict__ offs_k,
                                                       const int32_t* __restrict__ cnt,
                                                       const float* __restrict__ budget, double theta,
                                                       int rule, int per_row, int32_t* __restrict__ n_keep,
                                                       int32_t* __restrict__ n_rows) {
  __shared__ int s_sum[32], s_nq[32], s_nk[32], s_n, s_NK;
  const int bh = blockIdx.x, t = threadIdx.x;
  const int32_t* oq = offs_q + (size_t)bh * (kq + 1);
  const int32_t* ok = offs_k + (size_t)bh * (kk + 1);
  int sum = 0, nq = 0, nk = 0;
  for (int a = t; a < kq; a += 1024) {
    if (oq[a + 1] - oq[a] > 0) { ++nq; sum += cnt[(size_t)bh * kq + a]; }
  }
  for (int j = t; j < kk; j += 1024) nk += (ok[j + 1] - ok[j] > 0) ? 1 : 0;
  sum = warp_sum(sum); nq = warp_sum(nq); nk = warp_sum(nk);
  if ((t & 31) == 0) { s_sum[t >> 5] = sum; s_nq[t >> 5] = nq; s_nk[t >> 5] = nk; }
  __syncthreads();
  const double b = (double)budget[bh % H];
  if (t == 0) {
    int S = 0, NQ = 0, NK = 0;
    for (int w = 0; w < 32; ++w) { S += s_sum[w]; NQ += s_nq[w]; NK += s_nk[w]; }
    const int n_rec = NQ > 0 ? (S + NQ - 1) / NQ : 1;
    const int n = rule_n(n_rec, b, theta, rule, kk, NK);
    n_keep[bh] = n;
    s_n = n;
    s_NK = NK;
  }
  if (!n_rows) return;
  __syncthreads();
  for (int a = t; a < kq; a += 1024)
    n_rows[(size_t)bh * kq + a] = (per_row && oq[a + 1] - oq[a] > 0)
                                      ? rule_n(cnt[(size_t)bh * kq + a], b, theta, rule, kk, s_NK) : s_n;
}

// grid (kq, BH), block 256: kept row = first n of order, ascending
__global__ void __launch_bounds__(256) k_select_emit(int kq, int kk, const int32_t* __restrict__ order,
                                                     const int32_t* __restrict__ n_keep,
                                                     const int32_t* __restrict__ n_rows,
                                                     int32_t* __restrict__ kept) {
  __shared__ uint32_t flags[kMaxClusters / 32];
  __shared__ int sbuf[32];
  const int a = blockIdx.x, bh = blockIdx.y, t = threadIdx.x;
  const int n = n_rows ? n_rows[(size_t)bh * kq + a] : n_keep[bh];
  for (int w = t; w < kMaxClusters / 32; w += 256) flags[w] = 0u;
  __syncthreads();
  const int32_t* ord = order + ((size_t)bh * kq + a) * kk;
  for (int i = t; i < n; i += 256) {
    const int j = ord[i];
    atomicOr(&flags[j >> 5], 1u << (j & 31));
  }
  __syncthreads();
  // each thread owns 4 consecutive indices
  int c = 0;
  for (int u = 0; u < 4; ++u) {
    const int j = t * 4 + u;
    c += (j < kk && ((flags[j >> 5] >> (j & 31)) & 1u)) ? 1 : 0;
  }
  // block exclusive scan (256 threads)
  const int lane = t & 31, w = t >> 5;
  int x = c;
  for (int o = 1; o < 32; o <<= 1) { int y = __shfl_up_sync(0xffffffffu, x, o); if (lane >= o) x += y; }
  if (lane == 31) sbuf[w] = x;
  __syncthreads();
  int base = 0;
  for (int ww = 0; ww < w; ++ww) base += sbuf[ww];
  int pos = base + x - c;
  int32_t* out = kept + ((size_t)bh * kq + a) * kk;
  for (int u = 0; u < 4; ++u) {
    const int j = t * 4 + u;
    if (j < kk && ((flags[j >> 5] >> (j & 31)) & 1u)) out[pos++] = j;
  }
}

// grid BH, block 1024 (kq <= 1024): item_start[bh][a] (pairs of 128-row query tiles)
__global__ void __launch_bounds__(1024) k_worklist(int kq, const int32_t* __restrict__ offs_q,
                                                   int32_t* __restrict__ item_start) {
  extern __shared__ int sbuf_w[];
  const int bh = blockIdx.x, a = threadIdx.x;
  const int32_t* oq = offs_q + (size_t)bh * (kq + 1);
  int items = 0;
  if (a < kq) {
    const int len = oq[a + 1] - oq[a];
    const int tiles = (len + 127) / 128;
    items = (tiles + 1) / 2;
  }
  // block exclusive scan
  const int lane = a & 31, w = a >> 5;
  int x = items;
  for (int o = 1; o < 32; o <<= 1) { int y = __shfl_up_sync(0xffffffffu, x, o); if (lane >= o) x += y; }
  if (lane == 31) sbuf_w[w] = x;
  __syncthreads();
  int base = 0;
  for (int ww = 0; ww < w; ++ww) base += sbuf_w[ww];
  int32_t* is = item_start + (size_t)bh * (kq + 1);
  if (a < kq) is[a] = base + x - items;
  if (a == kq - 1) is[kq] = base + x;
}

int worklist_upper_bound(int N, int kq) { return (N + 255) / 256 + kq; }

cudaError_t launch_block_select(int BH, int H, int kq, int kk, int d, const float* cq,
                                const float* ck, const int32_t* offs_q, const int32_t* offs_k,
                                const float* budget, double tau, double theta, int rule, int flags,
                                int32_t* n_keep, int32_t* n_rows, int32_t* kept, int32_t* order,
                                int32_t* cnt, double* abar, cudaStream_t st) {
  const int weighted = (flags & 2) ? 1 : 0;
  const int need_cnt = rule != 2;  // FIXED (rule 2): n = n_b for every row, the recall counts are unused
  int P2 = 256;
  while (P2 < kk) P2 <<= 1;
  const size_t smem = (size_t)P2 * 16 + (size_t)P2 * 4;
  const dim3 gab((kk + 63) / 64, (kq + 63) / 64, BH);
  constexpr int sab = 2 * 64 * 65 * 8;  // > 48 KB: opt in
  if (d == 128) {
    cudaError_t e = cudaFuncSetAttribute(k_abar<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, sab);
    if (e != cudaSuccess) return e;
    k_abar<128><<<gab, 256, sab, st>>>(kq, kk, cq, ck, abar);
  } else {
    cudaError_t e = cudaFuncSetAttribute(k_abar<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, sab);
    if (e != cudaSuccess) return e;
    k_abar<64><<<gab, 256, sab, st>>>(kq, kk, cq, ck, abar);
  }
  if (P2 == 256)
    k_select_rows<1><<<dim3(kq, BH), 256, smem, st>>>(kq, kk, d, abar, offs_q, offs_k, tau, weighted, need_cnt, order, cnt);
  else if (P2 == 512)
    k_select_rows<2><<<dim3(kq, BH), 256, smem, st>>>(kq, kk, d, abar, offs_q, offs_k, tau, weighted, need_cnt, order, cnt);
  else
    k_select_rows<4><<<dim3(kq, BH), 256, smem, st>>>(kq, kk, d, abar, offs_q, offs_k, tau, weighted, need_cnt, order, cnt);
  k_select_count<<<BH, 1024, 0, st>>>(H, kq, kk, offs_q, offs_k, cnt, budget, theta, rule, flags & 1, n_keep,
                                      n_rows);
  k_select_emit<<<dim3(kq, BH), 256, 0, st>>>(kq, kk, order, n_keep, n_rows, kept);
  return cudaGetLastError();
}

cudaError_t launch_worklist(int BH, int kq, const int32_t* offs_q, int32_t* item_start,
                            cudaStream_t st) {
  const int threads = ((kq + 31) / 32) * 32;
  k_worklist<<<BH, threads, 32 * sizeof(int), st>>>(kq, offs_q, item_start);
  return cudaGetLastError();
}

}  // namespace cs
