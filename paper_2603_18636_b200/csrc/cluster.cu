// cluster.cu — co-clustering support kernels for Alg. 1 on sm_100a:
//   k_init_sample   : Sample(X, K) (R4) + C^(0) = X[idx]
//   k_gamma         : Gamma = C_a^T C_a (fp64)               } anchor prep for the reduced-form
//   k_anchor_w      : W_j = Gamma c_j / ||c_j C_a^T|| -> bf16 } assignment (a2)
//                     hi/lo split
//   k_seg_mean      : C_j = mean of the members of cluster j, optional permuted copy
//   k_csort_*       : stable counting sort labels -> perm, offs (implied by P:1266)
//   k_permute_rows  : x_perm[p] = x[perm[p]]
#include "kernels.cuh"

namespace cs {

// ---------------------------------------------------------------------------------------------
// block-wide exclusive scan (int), blockDim.x multiple of 32, <= 1024
// ---------------------------------------------------------------------------------------------
__device__ int block_exclusive_scan(int v, int* total, int* sbuf /*[32]*/) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sbuf[w] = x;
  __syncthreads();
  if (w == 0) {
    int s = lane < nw ? sbuf[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    sbuf[lane] = s;  // inclusive warp totals
  }
  __syncthreads();
  int base = w > 0 ? sbuf[w - 1] : 0;
  if (total) *total = sbuf[nw - 1];
  int r = base + x - v;
  __syncthreads();
  return r;
}

// ---------------------------------------------------------------------------------------------
// a1: init sampling.  grid (BH, 2 sides), block 256, dyn smem = bitmap words + idx[K]
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_init_sample(XView q, XView k, int N, int d, int kq, int kk,
                                                     unsigned long long seed, int h_off, int h_tot,
                                                     const int32_t* __restrict__ init_q,
                                                     const int32_t* __restrict__ init_k,
                                                     float* __restrict__ cq, float* __restrict__ ck) {
  extern __shared__ uint32_t sm_bits[];
  __shared__ int sbuf[32];
  // grid (BH, 2 sides, G): every CTA of a (bh, side) draws the same (deterministic) sample and
  // gathers its own 1/G of the K centroid rows, so the gather is spread over many SMs
  const int bh = blockIdx.x, side = blockIdx.y;
  const int K = side ? kk : kq;
  const int32_t* init = side ? init_k : init_q;
  const XView X = side ? k : q;
  float* C = (side ? ck : cq) + (size_t)bh * K * d;
  const int nwords = (N + 31) >> 5;
  int* idx = reinterpret_cast<int*>(sm_bits + ((nwords + 3) & ~3));  // 16-byte aligned (int4 loads)
  if (init) {
    for (int j = threadIdx.x; j < K; j += blockDim.x) idx[j] = init[(size_t)bh * K + j];
  } else {
    for (int w = threadIdx.x; w < nwords; w += blockDim.x) sm_bits[w] = 0u;
    // R4: splitmix64 stream, Floyd's algorithm.  The draws do not depend on the chosen set
    // (draw i uses state seed + (i+1) * golden), so all K of them are computed in parallel:
    // t_i = next_i % (N - K + i + 1), staged in idx[]; only the set-insertion pass is serial.
    const long long key = (long long)(bh / X.H) * h_tot + h_off + bh % X.H;  // b*Ht + hg
    const unsigned long long s0 = seed ^ ((unsigned long long)(key * 2 + side) * 0x9E3779B97F4A7C15ull);
    for (int i = threadIdx.x; i < K; i += blockDim.x) {
      unsigned long long z = s0 + (unsigned long long)(i + 1) * 0x9E3779B97F4A7C15ull;
      z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
      z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
      z ^= z >> 31;
      idx[i] = (int)(z % (unsigned long long)(N - K + i + 1));
    }
    __syncthreads();
    // Floyd's insertions, resolved in parallel (identical picks): with j_i = N - K + i,
    //  - t_i < N - K: t_i was picked before iff an earlier draw has the same value (the first
    //    occurrence of a value below N - K is always picked), so pick_i = dup ? j_i : t_i;
    //  - t_i == j_i: never picked before -> pick_i = t_i;
    //  - N - K <= t_i < j_i (t_i = j_m, m < i; about K^2 / 2N draws): j_m was picked before iff
    //    pick_m == j_m or an earlier draw t_k == j_m (m <= k < i) was picked as itself; resolved by
    //    one thread in increasing i over just these draws.
    int* pick = idx + K;            // [K]
    uint32_t* caseb = reinterpret_cast<uint32_t*>(pick + K);  // [32] bitmap of the third case
    const int NK = N - K;
    for (int w = threadIdx.x; w < 32; w += blockDim.x) caseb[w] = 0u;
    __syncthreads();
    for (int i = threadIdx.x; i < K; i += blockDim.x) {
      const int t = idx[i];
      if (t < NK) {
        // branch-free scan of the earlier draws, 4 per broadcast 16-byte load (every lane of the
        // warp reads the same addresses in the same iteration)
        int dup = 0, k2 = 0;
        for (; k2 + 4 <= i; k2 += 4) {
          const int4 v = *reinterpret_cast<const int4*>(idx + k2);
          dup |= (v.x == t) | (v.y == t) | (v.z == t) | (v.w == t);
        }
        for (; k2 < i; ++k2) dup |= idx[k2] == t;
        pick[i] = dup ? NK + i : t;
      } else if (t == NK + i) {
        pick[i] = t;
      } else {
        pick[i] = -1;
        atomicOr(&caseb[i >> 5], 1u << (i & 31));
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 0; w < 32; ++w) {
        uint32_t mb = caseb[w];
        while (mb) {
          const int i = (w << 5) + __ffs(mb) - 1;
          mb &= mb - 1;
          const int t = idx[i], m = t - NK;
          bool taken = pick[m] == t;  // j_m picked at step m
          for (int w2 = m >> 5; w2 <= (i >> 5) && !taken; ++w2) {  // earlier third-case draws == j_m
            uint32_t mk = caseb[w2];
            while (mk && !taken) {
              const int k2 = (w2 << 5) + __ffs(mk) - 1;
              mk &= mk - 1;
              if (k2 >= m && k2 < i && idx[k2] == t && pick[k2] == t) taken = true;
            }
          }
          pick[i] = taken ? NK + i : t;
        }
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < K; i += blockDim.x) atomicOr(&sm_bits[pick[i] >> 5], 1u << (pick[i] & 31));
    __syncthreads();
    // ascending compaction of the bitmap: each thread owns a contiguous word range
    const int per = (nwords + blockDim.x - 1) / blockDim.x;
    const int w0 = threadIdx.x * per, w1 = min(nwords, w0 + per);
    int cnt = 0;
    for (int w = w0; w < w1; ++w) cnt += __popc(sm_bits[w]);
    int pos = block_exclusive_scan(cnt, nullptr, sbuf);
    for (int w = w0; w < w1; ++w) {
      uint32_t m = sm_bits[w];
      while (m) {
        int b = __ffs(m) - 1;
        m &= m - 1;
        idx[pos++] = (w << 5) + b;
      }
    }
  }
  __syncthreads();
  // C^(0)[j] = X[idx[j]]  (bf16 -> fp32): 8 bf16 (16 B) per thread and load; 4 independent loads
  // in flight per thread before the converts / stores (one launch per layer: latency matters)
  const int b = bh / X.H, h = bh % X.H;
  const int vpr = d / 8;  // 16-byte vectors per row
  const int per = (K + gridDim.z - 1) / gridDim.z;
  const int jbeg = min(K, (int)blockIdx.z * per), jend = min(K, jbeg + per);
  const int total = jend * vpr;
  for (int e0 = jbeg * vpr + threadIdx.x; e0 < total; e0 += 4 * blockDim.x) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = e0 + u * blockDim.x;
      if (e < total) v[u] = *reinterpret_cast<const uint4*>(X.row(b, h, idx[e / vpr]) + (e % vpr) * 8);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = e0 + u * blockDim.x;
      if (e >= total) break;
      const int j = e / vpr, c = (e % vpr) * 8;
      const __nv_bfloat16* pv = reinterpret_cast<const __nv_bfloat16*>(&v[u]);
      float4 lo, hi;
      lo.x = __bfloat162float(pv[0]); lo.y = __bfloat162float(pv[1]); lo.z = __bfloat162float(pv[2]); lo.w = __bfloat162float(pv[3]);
      hi.x = __bfloat162float(pv[4]); hi.y = __bfloat162float(pv[5]); hi.z = __bfloat162float(pv[6]); hi.w = __bfloat162float(pv[7]);
      float4* dst = reinterpret_cast<float4*>(C + (size_t)j * d + c);
      dst[0] = lo;
      dst[1] = hi;
    }
  }
}

// Anchor-prep arithmetic type.  fp32 (default): Gamma sums K_a <= 1024 products and W_j = Gamma c_j
// 128 more, so W carries ~1e-6 relative error, below the 2^-17 resolution of its bf16 hi + lo split
// that the assignment GEMM consumes; fp64 (-DCS_PREP_FP64) for A/B comparisons.
#ifdef CS_PREP_FP64
typedef double prep_t;
typedef double2 prep2_t;
__device__ __forceinline__ __nv_bfloat16 to_bf16(double v) { return __double2bfloat16(v); }
#else
typedef float prep_t;
typedef float2 prep2_t;
__device__ __forceinline__ __nv_bfloat16 to_bf16(float v) { return __float2bfloat16_rn(v); }
#endif

// ---------------------------------------------------------------------------------------------
// a2: Gamma = C_a^T C_a (prep_t: fp32 by default, fp64 with -DCS_PREP_FP64).  grid (BH, NB (NB+1) / 2), block 256: one 64 x 64 block of the
// upper triangle of Gamma per CTA (an off-diagonal block also writes its mirror: Gamma is
// symmetric); thread (ti, tj) = (t / 16, t % 16) owns the 4 x 4 outputs (e0 + ti + 16 i,
// f0 + tj + 16 j): the 16 lanes of a half-warp read 16 consecutive elements (one wavefront for fp64) and
// the two halves the same ones (broadcast).
// Rows of C_a are staged in fp64 chunks of 32; per staged row 8 LDS.64 feed 16 DFMA.
// ---------------------------------------------------------------------------------------------
template <int D, int TB>
__global__ void __launch_bounds__(256) k_gamma(const float* __restrict__ ca, int ka,
                                               prep_t* __restrict__ gamma) {
  // split over the anchor rows: CTA z sums rows [z GR, (z+1) GR) into the partial Gamma_z (a
  // [gridDim.z][BH][D][D] slab); k_gamma_reduce adds the partials into slab 0 in a fixed order.
  // Short serial loops keep the kernel off the latency floor when few heads share a launch
  // (head-parallel ranks).
  constexpr int CH = 32, NB = D / TB, GR = kGammaRows, RT = TB / 16;  // RT x RT outputs per thread
  __shared__ __align__(16) prep_t sa[CH][D];
  // upper-triangle block index -> (row block, column block), column block >= row block
  int rb = 0, cb = blockIdx.y;
  while (cb >= NB - rb) { cb -= NB - rb; ++rb; }
  cb += rb;
  const int bh = blockIdx.x, e0 = rb * TB, f0 = cb * TB;
  const int r_beg = blockIdx.z * GR, r_end = min(ka, r_beg + GR);
  const float* A = ca + (size_t)bh * ka * D;
  gamma += (size_t)blockIdx.z * gridDim.x * D * D;
  const int t = threadIdx.x, ti = t >> 4, tj = t & 15;
  prep_t acc[RT][RT];
#pragma unroll
  for (int i = 0; i < RT; ++i)
#pragma unroll
    for (int j = 0; j < RT; ++j) acc[i][j] = prep_t(0);
  for (int a0 = r_beg; a0 < r_end; a0 += CH) {
    const int n = min(CH, r_end - a0);
    __syncthreads();
    for (int i = t; i < CH * D / 4; i += 256) {
      const int r = i / (D / 4), c = (i % (D / 4)) * 4;
      float4 v = r < n ? *reinterpret_cast<const float4*>(A + (size_t)(a0 + r) * D + c) : make_float4(0.f, 0.f, 0.f, 0.f);
      sa[r][c] = v.x; sa[r][c + 1] = v.y; sa[r][c + 2] = v.z; sa[r][c + 3] = v.w;
    }
    __syncthreads();
    for (int r = 0; r < n; ++r) {
      prep_t ve[RT], vf[RT];
#pragma unroll
      for (int i = 0; i < RT; ++i) { ve[i] = sa[r][e0 + ti + 16 * i]; vf[i] = sa[r][f0 + tj + 16 * i]; }
#pragma unroll
      for (int i = 0; i < RT; ++i)
#pragma unroll
        for (int j = 0; j < RT; ++j) acc[i][j] = fma(ve[i], vf[j], acc[i][j]);
    }
  }
  prep_t* G = gamma + (size_t)bh * D * D;
#pragma unroll
  for (int i = 0; i < RT; ++i)
#pragma unroll
    for (int j = 0; j < RT; ++j) G[(size_t)(e0 + ti + 16 * i) * D + f0 + tj + 16 * j] = acc[i][j];
  if (rb != cb) {
#pragma unroll
    for (int i = 0; i < RT; ++i)
#pragma unroll
      for (int j = 0; j < RT; ++j) G[(size_t)(f0 + tj + 16 * j) * D + e0 + ti + 16 * i] = acc[i][j];
  }
}

// slab 0 += slabs 1 .. nparts-1 (fixed order: deterministic); grid ceil(BH D D / 2 / 256)
__global__ void __launch_bounds__(256) k_gamma_reduce(prep_t* __restrict__ gamma, size_t slab, int nparts) {
  const size_t i = ((size_t)blockIdx.x * 256 + threadIdx.x) * 2;
  if (i >= slab) return;
  prep2_t a = *reinterpret_cast<const prep2_t*>(gamma + i);
  for (int z = 1; z < nparts; ++z) {
    const prep2_t b = *reinterpret_cast<const prep2_t*>(gamma + (size_t)z * slab + i);
    a.x += b.x;
    a.y += b.y;
  }
  *reinterpret_cast<prep2_t*>(gamma + i) = a;
}

// ---------------------------------------------------------------------------------------------
// a2: w_j = Gamma c_j (= (C_s Gamma)_j, Gamma symmetric), n_j^2 = ||c_j C_a^T||^2 = c_j . w_j,
//     W_j = w_j / n_j  ->  Wsplit[bh][j] = [bf16(W) | bf16(W - bf16(W))]
// grid (ks_pad / 32, BH), block 256, dyn smem 2 * 32 * D prep_t: 32 centroids per CTA.
// Thread (tj, te): centroids j0 + JPT tj .. +JPT-1, output columns te + EG e, e < 4 (EG = D/4;
// consecutive lanes read consecutive Gamma columns).  Gamma is streamed through shared memory in chunks of 32 rows.  Rows j >= ks
// are written as zeros (padding).
// ---------------------------------------------------------------------------------------------
template <int D, int J>
__global__ void __launch_bounds__(256) k_anchor_w(const float* __restrict__ cs_, int ks, int ks_pad,
                                                  const prep_t* __restrict__ gamma,
                                                  __nv_bfloat16* __restrict__ wsplit) {
  constexpr int EG = D / 4, JG = 256 / EG, JPT = J / JG, FCH = 32;
  static_assert(JPT >= 1, "at least one centroid per thread");
  extern __shared__ __align__(16) prep_t sm_aw[];
  prep_t (*sc)[D] = reinterpret_cast<prep_t (*)[D]>(sm_aw);           // [J][D]   centroids
  prep_t (*sg)[D] = reinterpret_cast<prep_t (*)[D]>(sm_aw + J * D);   // [FCH][D] Gamma rows
  const int bh = blockIdx.y, j0 = blockIdx.x * J, t = threadIdx.x;
  const int te = t % EG, tj = t / EG;
  const float* S = cs_ + (size_t)bh * ks * D;
  const prep_t* G = gamma + (size_t)bh * D * D;
  for (int i = t; i < J * D / 4; i += 256) {
    const int r = i / (D / 4), c = (i % (D / 4)) * 4;
    float4 v = (j0 + r < ks) ? *reinterpret_cast<const float4*>(S + (size_t)(j0 + r) * D + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    sc[r][c] = v.x; sc[r][c + 1] = v.y; sc[r][c + 2] = v.z; sc[r][c + 3] = v.w;
  }
  prep_t w[JPT][4];
#pragma unroll
  for (int i = 0; i < JPT; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) w[i][e] = prep_t(0);
  for (int f0 = 0; f0 < D; f0 += FCH) {
    __syncthreads();
    for (int i = t; i < FCH * D / 2; i += 256) {
      const int r = i / (D / 2), c = (i % (D / 2)) * 2;
      const prep2_t g = *reinterpret_cast<const prep2_t*>(G + (size_t)(f0 + r) * D + c);
      sg[r][c] = g.x; sg[r][c + 1] = g.y;
    }
    __syncthreads();
#pragma unroll 4
    for (int f = 0; f < FCH; ++f) {
      prep_t g[4], c[JPT];
#pragma unroll
      for (int e = 0; e < 4; ++e) g[e] = sg[f][te + EG * e];
#pragma unroll
      for (int i = 0; i < JPT; ++i) c[i] = sc[JPT * tj + i][f0 + f];
#pragma unroll
      for (int i = 0; i < JPT; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) w[i][e] = fma(g[e], c[i], w[i][e]);
    }
  }
  // n_j^2 = sum_e c_j[e] w_j[e]: partial over this thread's 4 columns, reduced over the EG
  // threads of the centroid group (consecutive lanes) in a fixed butterfly order
#pragma unroll
  for (int i = 0; i < JPT; ++i) {
    const int jl = JPT * tj + i, j = j0 + jl;
    prep_t n2 = prep_t(0);
#pragma unroll
    for (int e = 0; e < 4; ++e) n2 = fma(sc[jl][te + EG * e], w[i][e], n2);
#pragma unroll
    for (int o = EG / 2; o > 0; o >>= 1) n2 += __shfl_xor_sync(0xffffffffu, n2, o);
    if (j >= ks_pad) continue;
    __nv_bfloat16* out = wsplit + ((size_t)bh * ks_pad + j) * (2 * D);
    __nv_bfloat16 hi[4], lo[4];
    if (j < ks) {
      const prep_t inv = n2 > prep_t(0) ? prep_t(1) / sqrt(n2) : prep_t(0);  // ||Pbar_j|| = 0 -> W_j = 0
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const prep_t wv = w[i][e] * inv;
        hi[e] = to_bf16(wv);
        lo[e] = to_bf16(wv - (prep_t)__bfloat162float(hi[e]));
      }
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) { hi[e] = __float2bfloat16(0.f); lo[e] = __float2bfloat16(0.f); }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) { out[te + EG * e] = hi[e]; out[D + te + EG * e] = lo[e]; }
  }
}

// ---------------------------------------------------------------------------------------------
// k-means baseline (NEXT-2, "w/o On" P:1058): L(i) = argmin_j ||x_i - c_j|| = argmax_j x_i.c_j -
// ||c_j||^2/2 -> the same assignment GEMM with W_j = c_j (bf16 hi + lo) and a bias epilogue.
// grid (ks_pad / 8, BH), block 256: one warp per centroid.
// ---------------------------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(256) k_kmeans_w(const float* __restrict__ cs_, int ks, int ks_pad,
                                                  __nv_bfloat16* __restrict__ wsplit, float* __restrict__ bias) {
  constexpr int PL = D / 32;  // columns per lane
  const int bh = blockIdx.y, j = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (j >= ks_pad) return;
  __nv_bfloat16* out = wsplit + ((size_t)bh * ks_pad + j) * (2 * D);
  double n2 = 0.0;
#pragma unroll
  for (int i = 0; i < PL; ++i) {
    const int e = lane + 32 * i;
    const float c = j < ks ? cs_[((size_t)bh * ks + j) * D + e] : 0.f;
    const __nv_bfloat16 hi = __float2bfloat16(c);
    out[e] = hi;
    out[D + e] = __float2bfloat16(c - __bfloat162float(hi));
    n2 = fma((double)c, (double)c, n2);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) n2 += __shfl_xor_sync(0xffffffffu, n2, o);
  if (lane == 0) bias[(size_t)bh * ks_pad + j] = j < ks ? (float)(-0.5 * n2) : 0.f;
}

cudaError_t launch_kmeans_prep(const float* cself, int ks, int ks_pad, int BH, int d, __nv_bfloat16* wsplit,
                               float* bias, cudaStream_t st) {
  const dim3 grid((ks_pad + 7) / 8, BH);
  if (d == 128)
    k_kmeans_w<128><<<grid, 256, 0, st>>>(cself, ks, ks_pad, wsplit, bias);
  else
    k_kmeans_w<64><<<grid, 256, 0, st>>>(cself, ks, ks_pad, wsplit, bias);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// a5/a7: centroid update.  grid (ceil(K / CPB), BH), block 32 NWC CPB threads: CPB clusters per
// CTA (1 by default: a CTA's warps never wait at the final barrier for a larger cluster sharing
// the CTA) with NWC warps each (NWC from the mean cluster size, so small clusters do not leave
// most of a CTA idle).  Warp ws of a cluster sums a contiguous chunk of its sorted positions;
// fixed order -> deterministic.  Empty cluster: untouched (R5).
// ---------------------------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(256) k_seg_mean(XView x, int N, int K, int nwc,
                                                  const int32_t* __restrict__ perm,
                                                  const int32_t* __restrict__ offs,
                                                  float* __restrict__ C,
                                                  __nv_bfloat16* __restrict__ xperm) {
  constexpr int LPR = D / 8;        // lanes per row: 16-byte (8 x bf16) vector per lane
  constexpr int RPW = 32 / LPR;     // rows per warp instruction (2 or 4)
#ifndef CS_SEG_U
#define CS_SEG_U 8
#endif
  constexpr int NWMAX = 8, U = CS_SEG_U;  // warps (at most), rows in flight per lane group
  __shared__ float part[NWMAX * RPW][D];
  const int bh = blockIdx.y;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, NW = blockDim.x >> 5;
  const int cpb = NW / nwc, cl = w / nwc, ws = w % nwc;
  const int j = blockIdx.x * cpb + cl;
  const int grp = lane / LPR, gl = lane % LPR;  // row group inside the warp, lane inside the row
  const int32_t* of = offs + (size_t)bh * (K + 1);
  const int beg = j < K ? of[j] : 0, end = j < K ? of[j + 1] : 0, cnt = end - beg;
  const int b = bh / x.H, h = bh % x.H;
  // fixed partition of the cluster's positions: warp ws owns a contiguous chunk, row group grp
  // takes every RPW-th position of it -> deterministic summation order
  const int chunk = (cnt + nwc - 1) / nwc;
  const int p0 = beg + ws * chunk, p1 = min(end, p0 + chunk);
  const int32_t* pm = perm + (size_t)bh * N;
  float acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = 0.f;
  for (int p = p0 + grp; p < p1; p += U * RPW) {
    uint4 v[U];
    int tok[U];
#pragma unroll
    for (int u = 0; u < U; ++u) tok[u] = (p + u * RPW < p1) ? pm[p + u * RPW] : -1;
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (tok[u] >= 0) v[u] = *reinterpret_cast<const uint4*>(x.row(b, h, tok[u]) + gl * 8);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (tok[u] < 0) break;
      const __nv_bfloat16* e = reinterpret_cast<const __nv_bfloat16*>(&v[u]);
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] += __bfloat162float(e[i]);
      if (xperm) *reinterpret_cast<uint4*>(xperm + ((size_t)bh * N + p + u * RPW) * D + gl * 8) = v[u];
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) part[w * RPW + grp][gl * 8 + i] = acc[i];
  __syncthreads();
  // cluster c of the CTA: partial rows [c nwc RPW, (c+1) nwc RPW), summed in a fixed order
  for (int o = threadIdx.x; o < cpb * D; o += blockDim.x) {
    const int c = o / D, col = o % D, jc = blockIdx.x * cpb + c;
    if (jc >= K) continue;
    const int n = of[jc + 1] - of[jc];
    if (n == 0) continue;
    float sum = 0.f;
    for (int q = 0; q < nwc * RPW; ++q) sum += part[c * nwc * RPW + q][col];
    C[((size_t)bh * K + jc) * D + col] = sum / (float)n;
  }
}

// ---------------------------------------------------------------------------------------------
// a4/a7: stable counting sort.  Tiles of kSortTile tokens.
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_csort_hist(const int32_t* __restrict__ lab, int N, int K,
                                                    int ntiles, int32_t* __restrict__ hist) {
  extern __shared__ int sh_hist[];
  const int bh = blockIdx.y, t = blockIdx.x;
  for (int c = threadIdx.x; c < K; c += blockDim.x) sh_hist[c] = 0;
  __syncthreads();
  const int i0 = t * kSortTile, i1 = min(N, i0 + kSortTile);
  const int32_t* L = lab + (size_t)bh * N;
  constexpr int RT = kSortTile / 256;  // labels per thread, all loads in flight before the atomics
  int lbl[RT];
#pragma unroll
  for (int r = 0; r < RT; ++r) {
    const int i = i0 + r * 256 + threadIdx.x;
    lbl[r] = i < i1 ? L[i] : -1;
  }
#pragma unroll
  for (int r = 0; r < RT; ++r)
    if (lbl[r] >= 0) atomicAdd(&sh_hist[lbl[r]], 1);
  __syncthreads();
  int32_t* H = hist + ((size_t)bh * ntiles + t) * K;
  for (int c = threadIdx.x; c < K; c += blockDim.x) H[c] = sh_hist[c];
}

// grid (ceil(K / 32), BH), block 256 = 32 labels x 8 tile groups: hist (counts) -> per-tile bases
// relative to the label's first position, in place; tot[bh][c] = label sizes.  The serial chains
// are ceil(ntiles / 8) long (not ntiles), so the kernel stays short when few heads share a launch.
__global__ void __launch_bounds__(256) k_csort_scan(int K, int ntiles, int32_t* __restrict__ hist,
                                                    int32_t* __restrict__ tot) {
  __shared__ int gs[8][33];
  const int bh = blockIdx.y, cl = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + cl;
  const int per = (ntiles + 7) / 8, t0 = g * per, t1 = min(ntiles, t0 + per);
  int32_t* H = hist + (size_t)bh * ntiles * K;
  int sum = 0;
  if (c < K)
    for (int t = t0; t < t1; ++t) sum += H[(size_t)t * K + c];
  gs[g][cl] = sum;
  __syncthreads();
  int base = 0;
  for (int q = 0; q < g; ++q) base += gs[q][cl];
  if (c < K) {
    for (int t = t0; t < t1; ++t) {
      const int h = H[(size_t)t * K + c];
      H[(size_t)t * K + c] = base;
      base += h;
    }
    if (g == 7) tot[(size_t)bh * K + c] = base;
  }
}

// grid (ntiles, BH), block 256 = 8 warps x 128 tokens of one tile, dyn smem 9 K ints.
// Label starts = exclusive scan of tot (every CTA, K <= 1024; CTA 0 also writes offs); per-warp
// label counts (match_any) -> per-warp cursors -> each warp scatters its tokens in order: stable.
__global__ void __launch_bounds__(256) k_csort_scatter(const int32_t* __restrict__ lab, int N, int K,
                                                       int ntiles, const int32_t* __restrict__ base,
                                                       const int32_t* __restrict__ tot,
                                                       int32_t* __restrict__ offs,
                                                       int32_t* __restrict__ perm) {
  extern __shared__ int sh_cs[];
  int* lstart = sh_cs;      // [K]
  int* wc = sh_cs + K;      // [8][K]: per-warp counts, then per-warp cursors
  __shared__ int sbuf[32];
  const int bh = blockIdx.y, t = blockIdx.x, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // label starts
  const int per = (K + 255) / 256, c0 = threadIdx.x * per, c1 = min(K, c0 + per);
  const int32_t* T = tot + (size_t)bh * K;
  int loc = 0;
  for (int c = c0; c < c1; ++c) loc += T[c];
  int run = block_exclusive_scan(loc, nullptr, sbuf);
  for (int c = c0; c < c1; ++c) {
    lstart[c] = run;
    if (t == 0) offs[(size_t)bh * (K + 1) + c] = run;
    run += T[c];
  }
  if (t == 0 && threadIdx.x == 0) offs[(size_t)bh * (K + 1) + K] = N;
  for (int i = threadIdx.x; i < 8 * K; i += 256) wc[i] = 0;
  __syncthreads();
  const int32_t* L = lab + (size_t)bh * N;
  const int i0 = t * kSortTile + w * (kSortTile / 8), i1 = min(N, i0 + kSortTile / 8);
  const unsigned lt = (1u << lane) - 1u;
  int* cw = wc + w * K;
  // the warp's kSortTile / 8 labels, loaded once (all in flight together) for both passes;
  // out-of-range slots get unique negative dummy keys
  constexpr int RW = kSortTile / 8 / 32;
  int lbl[RW];
#pragma unroll
  for (int r = 0; r < RW; ++r) {
    const int me = i0 + r * 32 + lane;
    lbl[r] = me < i1 ? L[me] : -1 - lane;
  }
#pragma unroll
  for (int r = 0; r < RW; ++r) {  // per-warp label counts
    const int l = lbl[r];
    const unsigned peers = __match_any_sync(0xffffffffu, l);
    if (l >= 0 && __popc(peers & lt) == 0) cw[l] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  const int32_t* B0 = base + ((size_t)bh * ntiles + t) * K;
  for (int c = threadIdx.x; c < K; c += 256) {  // counts -> cursors
    int cur = lstart[c] + B0[c];
    for (int q = 0; q < 8; ++q) {
      const int n = wc[q * K + c];
      wc[q * K + c] = cur;
      cur += n;
    }
  }
  __syncthreads();
  int32_t* P = perm + (size_t)bh * N;
#pragma unroll
  for (int r = 0; r < RW; ++r) {
    const int me = i0 + r * 32 + lane;
    const int l = lbl[r];
    const bool valid = l >= 0;
    const unsigned peers = __match_any_sync(0xffffffffu, l);
    const int rank = __popc(peers & lt);
    const int basep = valid ? cw[l] : 0;
    __syncwarp();
    if (valid) {
      P[basep + rank] = me;
      if (rank == 0) cw[l] = basep + __popc(peers);
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------------------------
// x_perm[bh][p][:] = x[b,h,perm[bh][p],:].  grid (ceil(N/16), BH), block 256 (16 rows / block)
// ---------------------------------------------------------------------------------------------
#ifndef CS_PERM_U
#define CS_PERM_U 4
#endif
constexpr int kPermU = CS_PERM_U;  // rows per thread: kPermU 16-byte loads in flight
__global__ void __launch_bounds__(256) k_permute_rows(XView x, int N, int d,
                                                      const int32_t* __restrict__ perm,
                                                      __nv_bfloat16* __restrict__ xp) {
  const int bh = blockIdx.y;
  const int lanes_per_row = d / 8;  // 16-byte chunks per row
  const int rows_per_pass = 256 / lanes_per_row;
  const int r = threadIdx.x / lanes_per_row, c = threadIdx.x % lanes_per_row;
  const int p0 = blockIdx.x * rows_per_pass * kPermU + r;
  const int b = bh / x.H, h = bh % x.H;
  int tok[kPermU];
  uint4 v[kPermU];
#pragma unroll
  for (int u = 0; u < kPermU; ++u) {
    const int p = p0 + u * rows_per_pass;
    tok[u] = p < N ? perm[(size_t)bh * N + p] : -1;
  }
#pragma unroll
  for (int u = 0; u < kPermU; ++u)
    if (tok[u] >= 0) v[u] = *reinterpret_cast<const uint4*>(x.row(b, h, tok[u]) + c * 8);
#pragma unroll
  for (int u = 0; u < kPermU; ++u)
    if (tok[u] >= 0)
      *reinterpret_cast<uint4*>(xp + ((size_t)bh * N + p0 + u * rows_per_pass) * d + c * 8) = v[u];
}

// ---------------------------------------------------------------------------------------------
// host-side launchers
// ---------------------------------------------------------------------------------------------
cudaError_t launch_init_sample(XView q, XView k, int BH, int N, int d, int kq, int kk,
                               unsigned long long seed, int h_off, int h_tot, const int32_t* init_q,
                               const int32_t* init_k, float* cq, float* ck, cudaStream_t st) {
  const size_t smem = (size_t)(((N + 31) / 32 + 3) & ~3) * 4 + (size_t)max(kq, kk) * 8 + 32 * 4;  // bitmap, draws, picks, flags
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_init_sample, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
  }
  // gather parts per (bh, side): about two CTAs per SM in total (the sampling is recomputed per
  // part: ~K^2/4 broadcast compares, cheap next to the row gather it parallelises)
  int G = (2 * 148 + 2 * BH - 1) / (2 * BH);
  G = G < 1 ? 1 : (G > 16 ? 16 : G);
  k_init_sample<<<dim3(BH, 2, G), 256, smem, st>>>(q, k, N, d, kq, kk, seed, h_off, h_tot, init_q, init_k,
                                                   cq, ck);
  return cudaGetLastError();
}

// Output tiling of the two prep kernels: Gamma in 64 x 64 blocks and W in 32 centroids per CTA, or
// finer tiles when a launch would not fill one wave of the SMs (few heads per call: head-parallel
// ranks, small models).  Every output keeps its own sequential summation order, so the choice
// does not change a single bit (and head-sharded calls stay bit-equal to unsharded ones).
cudaError_t launch_anchor_prep(const float* ca, int ka, const float* cself, int ks, int ks_pad,
                               int BH, int d, void* gamma_ws, __nv_bfloat16* wsplit, cudaStream_t st) {
  prep_t* gamma = static_cast<prep_t*>(gamma_ws);
  const int nparts = (ka + kGammaRows - 1) / kGammaRows;  // gamma holds nparts x BH x d x d
  const size_t slab = (size_t)BH * d * d;
  int num_sms = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
  if (num_sms <= 0) num_sms = 148;
  const int nb64 = d / 64, nb32 = d / 32;
  const bool g_fine = BH * nparts * (nb64 * (nb64 + 1) / 2) < num_sms;  // 32 x 32 Gamma blocks
  const int jw = ((ks_pad + 31) / 32) * BH >= num_sms ? 32 : (((ks_pad + 15) / 16) * BH >= num_sms || d == 64 ? 16 : 8);
  auto launch_w = [&](auto kfn, int J) -> cudaError_t {
    const int smem = (J + 32) * d * (int)sizeof(prep_t);
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    kfn<<<dim3((ks_pad + J - 1) / J, BH), 256, smem, st>>>(cself, ks, ks_pad, gamma, wsplit);
    return cudaSuccess;
  };
  cudaError_t e;
  if (d == 128) {
    if (g_fine) k_gamma<128, 32><<<dim3(BH, nb32 * (nb32 + 1) / 2, nparts), 256, 0, st>>>(ca, ka, gamma);
    else k_gamma<128, 64><<<dim3(BH, nb64 * (nb64 + 1) / 2, nparts), 256, 0, st>>>(ca, ka, gamma);
    if (nparts > 1) k_gamma_reduce<<<(unsigned)((slab / 2 + 255) / 256), 256, 0, st>>>(gamma, slab, nparts);
    e = jw == 32 ? launch_w(k_anchor_w<128, 32>, 32) : jw == 16 ? launch_w(k_anchor_w<128, 16>, 16)
                                                                 : launch_w(k_anchor_w<128, 8>, 8);
  } else {
    if (g_fine) k_gamma<64, 32><<<dim3(BH, nb32 * (nb32 + 1) / 2, nparts), 256, 0, st>>>(ca, ka, gamma);
    else k_gamma<64, 64><<<dim3(BH, nb64 * (nb64 + 1) / 2, nparts), 256, 0, st>>>(ca, ka, gamma);
    if (nparts > 1) k_gamma_reduce<<<(unsigned)((slab / 2 + 255) / 256), 256, 0, st>>>(gamma, slab, nparts);
    e = jw == 32 ? launch_w(k_anchor_w<64, 32>, 32) : launch_w(k_anchor_w<64, 16>, 16);
  }
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_seg_mean(XView x, int BH, int N, int d, int K, const int32_t* perm,
                            const int32_t* offs, float* C, __nv_bfloat16* xperm, cudaStream_t st) {
  // warps per cluster: about one warp per CS_SEG_ROWS mean members, a power of two in [1, 8]
#ifndef CS_SEG_ROWS
#define CS_SEG_ROWS 64
#endif
  const int mean = N / K;
  int nwc = 1;
  while (nwc < 8 && nwc * CS_SEG_ROWS < mean) nwc <<= 1;
#ifndef CS_SEG_CPB
#define CS_SEG_CPB 1  // clusters per CTA: one, so a CTA's warps never wait for another cluster's rows
#endif
  const int cpb = CS_SEG_CPB * nwc > 8 ? 8 / nwc : CS_SEG_CPB;
  const dim3 grid((K + cpb - 1) / cpb, BH);
  const int threads = 32 * nwc * cpb;
  if (d == 128)
    k_seg_mean<128><<<grid, threads, 0, st>>>(x, N, K, nwc, perm, offs, C, xperm);
  else
    k_seg_mean<64><<<grid, threads, 0, st>>>(x, N, K, nwc, perm, offs, C, xperm);
  return cudaGetLastError();
}

cudaError_t launch_csort(const int32_t* lab, int BH, int N, int K, int32_t* perm, int32_t* offs,
                         int32_t* hist, cudaStream_t st) {
  const int ntiles = (N + kSortTile - 1) / kSortTile;
  int32_t* tot = hist + (size_t)BH * ntiles * K;  // label sizes [BH][K] after the tile histograms
  k_csort_hist<<<dim3(ntiles, BH), 256, K * sizeof(int), st>>>(lab, N, K, ntiles, hist);
  k_csort_scan<<<dim3((K + 31) / 32, BH), 256, 0, st>>>(K, ntiles, hist, tot);
  k_csort_scatter<<<dim3(ntiles, BH), 256, 9 * K * sizeof(int), st>>>(lab, N, K, ntiles, hist, tot, offs, perm);
  return cudaGetLastError();
}

cudaError_t launch_permute_rows(XView x, int BH, int N, int d, const int32_t* perm,
                                __nv_bfloat16* xp, cudaStream_t st) {
  const int rows_per_block = 256 / (d / 8) * kPermU;
  k_permute_rows<<<dim3((N + rows_per_block - 1) / rows_per_block, BH), 256, 0, st>>>(x, N, d, perm, xp);
  return cudaGetLastError();
}

}  // namespace cs

namespace cs {
// ---------------------------------------------------------------------------------------------
// Ulysses resharding helper: dst[b][a][:] = src[a][b][:] for rows of row_bytes (a multiple of 16)
// grid-stride over 16-byte vectors; coalesced reads and writes along the row.
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_block_transpose(int A, int B, int vpr, const uint4* __restrict__ src,
                                                         uint4* __restrict__ dst) {
  const long long total = (long long)A * B * vpr;
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < total; i += (long long)gridDim.x * 256) {
    const int v = (int)(i % vpr);
    const long long ab = i / vpr;
    const int b = (int)(ab % B), a = (int)(ab / B);
    dst[((long long)b * A + a) * vpr + v] = src[i];
  }
}

cudaError_t launch_block_transpose(int A, int B, size_t row_bytes, const void* src, void* dst, cudaStream_t st) {
  const int vpr = (int)(row_bytes / 16);
  const long long total = (long long)A * B * vpr;
  const int grid = (int)((total + 255) / 256 < 148 * 16 ? (total + 255) / 256 : 148 * 16);
  k_block_transpose<<<grid > 0 ? grid : 1, 256, 0, st>>>(A, B, vpr, static_cast<const uint4*>(src),
                                                          static_cast<uint4*>(dst));
  return cudaGetLastError();
}

// Ulysses in-bound pack (a13): T token blocks src_t [Nl, P * Hl, d] (rank-local tokens, all heads)
// -> dst [P, Nl, T, Hg, d] for the head group g (heads [g Hg, (g+1) Hg) of every rank's Hl-head
// block; Hg = Hl: all of them): chunk p (destination rank p) holds, per token, the T tensors' head
// rows side by side, so after ONE all_to_all_single the receiver sees [N, T, Hg, d] and tensor t is
// the strided [Hg, N, d] view (token stride T Hg d) the layer reads without a copy.
// vpr = 16-byte vectors per packed row (Hg d bf16), sstride / soff = vectors between consecutive
// (token, rank) rows of a source and the group's offset in such a row.
__global__ void __launch_bounds__(256) k_ulysses_pack(int Nl, int P, int T, int vpr, int sstride, int soff,
                                                      UlyssesSrcs srcs, uint4* __restrict__ dst) {
  const long long total = (long long)P * Nl * T * vpr;
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < total; i += (long long)gridDim.x * 256) {
    const int v = (int)(i % vpr);
    long long r = i / vpr;
    const int t = (int)(r % T);
    r /= T;
    const int n = (int)(r % Nl), p = (int)(r / Nl);
    dst[i] = srcs.p[t][((long long)n * P + p) * sstride + soff + v];
  }
}

cudaError_t launch_ulysses_pack(int Nl, int P, int T, size_t row_bytes, size_t src_row_bytes, size_t src_off_bytes,
                                const UlyssesSrcs& srcs, void* dst, cudaStream_t st) {
  const int vpr = (int)(row_bytes / 16);
  const long long total = (long long)P * Nl * T * vpr;
  const long long want = (total + 255) / 256;
  const int grid = (int)(want < 148 * 16 ? want : 148 * 16);
  k_ulysses_pack<<<grid > 0 ? grid : 1, 256, 0, st>>>(Nl, P, T, vpr, (int)(src_row_bytes / 16),
                                                      (int)(src_off_bytes / 16), srcs, static_cast<uint4*>(dst));
  return cudaGetLastError();
}
}  // namespace cs
