// assign.cu — Alg. 1 assignment (Step A: P:1214-1218, Step B: P:1222-1226) as a tcgen05 GEMM with
// a fused row-argmax epilogue, in the exact reduced form:
//     L(i) = argmin_j || Norm(x_i C_a^T) - Norm(c_j C_a^T) ||_2 = argmax_j x_i . W_j,
//     W_j  = (C_a^T C_a) c_j / ||c_j C_a^T||   (ties -> lowest j)
// W enters the tensor core as two bf16 parts (hi + lo): score = x_i.W_hi_j + x_i.W_lo_j,
// accumulated in fp32 over an inner dimension of 2d.
//
// Persistent kernel: one CTA per SM loops over work units = (head, 256 consecutive tokens = two
// 128-row tiles).  Per unit the centroid side is streamed in chunks of nch <= 128 columns
// (UMMA M=128, N=nch) through a 4-stage ring of 64-column W slabs; each slab feeds BOTH token
// tiles, halving W traffic from L2.  TMEM holds 2 buffers x 2 tiles x 128 fp32 columns, so the
// argmax epilogue of chunk c overlaps the MMAs of chunk c+1 (and of the next unit); X tiles are
// double-buffered across units.
// Warps 0-3: epilogue tile 0, 4-7: epilogue tile 1 (thread = token row = TMEM lane),
// warp 8: TMA producer, warp 9: TMEM allocator + MMA issuer.
// With a bias (the k-means baseline, NEXT-2: W_j = c_j, bias_j = -||c_j||^2 / 2, so argmax_j
// x.c_j - ||c_j||^2/2 = argmin_j ||x - c_j||) the epilogue adds bias[bh][j] before the argmax.
#include "kernels.cuh"

namespace cs {
namespace asg {

constexpr int BM = 128, TILES = 2, NSTW = 4, NTHREADS = 320, NCH_MAX = 128;
constexpr int WARP_PRODUCER = 8, WARP_MMA = 9;

template <int D>
struct Smem {
  static constexpr int HALVES = D / 64;
  static constexpr int XT = BM * D * 2;             // one 128-token tile
  static constexpr int HALF_X = BM * 128;
  static constexpr int XSTAGE = TILES * XT;         // one unit
  static constexpr int SLAB = NCH_MAX * 128;        // 64 columns x nch rows
  static constexpr int OFF_X = 0;
  static constexpr int OFF_W = OFF_X + 2 * XSTAGE;
  static constexpr int OFF_BAR = OFF_W + NSTW * SLAB;
  // x_full[2], x_empty[2], w_full[4], w_empty[4], acc_full[2], acc_empty[2]
  static constexpr int OFF_MISC = OFF_BAR + 8 * 16;
  static constexpr int BYTES = OFF_MISC + 16;
  static constexpr int ALLOC = BYTES + 1024;
};

// Grouped running argmax over 16 score columns j = jg .. jg+15 (columns >= ks are padding): a
// 3-input max tree (8 FMNMX) and one compare; the group that raised the running max is kept in
// registers and searched once per row at the end (argmax_finish).  Same result as a serial scan:
// exact fp32 compares, ties -> lowest index (strict > across groups, first equal element inside
// the winning group).
template <bool BIAS>
__device__ __forceinline__ void argmax_group(const uint32_t* v, const float* bs, int jg, int ks, float& best,
                                             int& best_j, float* keep) {
  float xs[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    xs[i] = __uint_as_float(v[i]);
    if constexpr (BIAS) xs[i] += bs[i];
  }
  if (jg + 16 > ks) {  // ragged last group (warp-uniform branch)
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (jg + i >= ks) xs[i] = -INFINITY;
  }
  const float m = fmaxf(fmax3(fmax3(xs[0], xs[1], xs[2]), fmax3(xs[3], xs[4], xs[5]), fmax3(xs[6], xs[7], xs[8])),
                        fmax3(fmax3(xs[9], xs[10], xs[11]), fmax3(xs[12], xs[13], xs[14]), xs[15]));
  const bool up = m > best;
  best = up ? m : best;
  best_j = up ? jg : best_j;
#pragma unroll
  for (int i = 0; i < 16; ++i) keep[i] = up ? xs[i] : keep[i];
}
__device__ __forceinline__ int argmax_finish(float best, int best_j, const float* keep) {
  int off = 15;
#pragma unroll
  for (int i = 15; i >= 0; --i) off = keep[i] == best ? i : off;
  return best_j + off;
}
// One pass over an accumulator chunk of nch columns (TMEM address t_acc, columns jbase ..), 16
// columns per TMEM load + wait (32 per wait with two loads in flight measured slower: 606 vs 559 us
// on the key side, more registers; the query side unchanged).
template <bool BIAS>
__device__ __forceinline__ void argmax_chunk(uint32_t t_acc, int nch, int jbase, int ks, const float* bias_row,
                                             float& best, int& best_j, float* keep) {
  for (int c0 = 0; c0 < nch; c0 += 16) {
    uint32_t v[16];
    float bs[16];
    tmem_ld16(t_acc + c0, v);
    if constexpr (BIAS) {  // warp-uniform address: broadcast loads
      const float4* b4 = reinterpret_cast<const float4*>(bias_row + jbase + c0);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float4 q = __ldg(b4 + i);
        bs[4 * i] = q.x; bs[4 * i + 1] = q.y; bs[4 * i + 2] = q.z; bs[4 * i + 3] = q.w;
      }
    }
    tmem_wait_ld();
    argmax_group<BIAS>(v, bs, jbase + c0, ks, best, best_j, keep);
  }
}

template <int D, bool BIAS>
__global__ void __launch_bounds__(NTHREADS, 1)
    k_assign(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_w,
             int H, int N, int ks, int nch, int ks_pad, int units_per_head, int num_units,
             const float* __restrict__ bias, int32_t* __restrict__ labels) {
  using L = Smem<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L::OFF_BAR);
  uint64_t* x_full = bars;
  uint64_t* x_empty = bars + 2;
  uint64_t* w_full = bars + 4;
  uint64_t* w_empty = bars + 4 + NSTW;
  uint64_t* acc_full = bars + 4 + 2 * NSTW;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + L::OFF_MISC);

  const int warp = warp_id(), lane = lane_id();
  const int nchunks = ks_pad / nch;
  // contiguous unit range per CTA: consecutive units mostly share the head, so when the whole
  // centroid side fits the W ring (one chunk) it stays resident in SMEM across units
  const int upc = (num_units + gridDim.x - 1) / gridDim.x;
  const int u_begin = blockIdx.x * upc, u_end = min(num_units, u_begin + upc);
  constexpr int SLABS = 2 * D / 64;  // 64-column slabs per chunk (hi halves then lo halves)

  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) { mbar_init(x_full + s, 1); mbar_init(x_empty + s, 1); }
    for (int s = 0; s < NSTW; ++s) { mbar_init(w_full + s, 1); mbar_init(w_empty + s, 1); }
    for (int t = 0; t < 2; ++t) { mbar_init(acc_full + t, 1); mbar_init(acc_empty + t, 2 * BM); }
    fence_barrier_init();
  }
  if (warp == WARP_MMA) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == WARP_PRODUCER) {
    if (lane == 0) {
      tma_prefetch_desc(&tm_x);
      tma_prefetch_desc(&tm_w);
      int g = 0;  // global slab counter
      int it = 0, prev_bh = -1;
      for (int u = u_begin; u < u_end; ++u, ++it) {
        const int bh = u / units_per_head, n0 = (u % units_per_head) * (TILES * BM);
        const int b = bh / H, h = bh % H;
        const int xs = it & 1;
        mbar_wait(x_empty + xs, ((it >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(x_full + xs, L::XSTAGE);
        for (int t = 0; t < TILES; ++t)
          for (int hf = 0; hf < L::HALVES; ++hf)
            tma_load_4d(sm + L::OFF_X + xs * L::XSTAGE + t * L::XT + hf * L::HALF_X, &tm_x, hf * 64,
                        n0 + t * BM, h, b, x_full + xs);
        const bool w_resident = nchunks == 1 && SLABS == NSTW && bh == prev_bh;
        for (int c = 0; c < nchunks; ++c)
          for (int s = 0; s < SLABS; ++s, ++g) {
            const int stage = g % NSTW;
            mbar_wait(w_empty + stage, ((g / NSTW) & 1) ^ 1);
            if (w_resident) {
              mbar_arrive(w_full + stage);  // same head, same slab already in this stage
            } else {
              mbar_arrive_expect_tx(w_full + stage, nch * 128);
              tma_load_2d(sm + L::OFF_W + stage * L::SLAB, &tm_w, s * 64, bh * ks_pad + c * nch,
                          w_full + stage);
            }
          }
        prev_bh = bh;
      }
    }
  } else if (warp == WARP_MMA) {
    if (lane == 0) {
      const uint32_t idesc = idesc_bf16(BM, nch, 0, 0);
      const uint32_t sX = smem_u32(sm + L::OFF_X), sW = smem_u32(sm + L::OFF_W);
      int g = 0, gc = 0, it = 0;
      for (int u = u_begin; u < u_end; ++u, ++it) {
        const int xs = it & 1;
        mbar_wait(x_full + xs, (it >> 1) & 1);
        for (int c = 0; c < nchunks; ++c, ++gc) {
          const int buf = gc & 1;
          mbar_wait(acc_empty + buf, ((gc >> 1) & 1) ^ 1);
          tc_fence_after();
          for (int s = 0; s < SLABS; ++s, ++g) {
            const int stage = g % NSTW;
            mbar_wait(w_full + stage, (g / NSTW) & 1);
            tc_fence_after();
            const int xh = s % L::HALVES;  // slab s pairs with x half (s mod halves)
#pragma unroll
            for (int t = 0; t < TILES; ++t) {
              const uint32_t d_tmem = tmem + (buf * TILES + t) * 128;
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const uint64_t ad = smem_desc_sw128(sX + xs * L::XSTAGE + t * L::XT + xh * L::HALF_X + k * 32, 16, 1024);
                const uint64_t bd = smem_desc_sw128(sW + stage * L::SLAB + k * 32, 16, 1024);
                mma_ss(d_tmem, ad, bd, idesc, (s > 0 || k > 0) ? 1u : 0u);
              }
            }
            mma_commit(w_empty + stage);
          }
          mma_commit(acc_full + buf);
        }
        mma_commit(x_empty + xs);
      }
    }
    __syncwarp();
  } else {
    // epilogue: running argmax over the valid centroid columns, ties -> lowest index
    const int t = warp >> 2, quad = warp & 3;
    const int r = quad * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    int gc = 0;
    for (int u = u_begin; u < u_end; ++u) {
      const int bh = u / units_per_head, n0 = (u % units_per_head) * (TILES * BM);
      float best = -INFINITY;
      int best_j = 0;
      float keep[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) keep[i] = -INFINITY;
      const float* bias_row = BIAS ? bias + (size_t)bh * ks_pad : nullptr;
      for (int c = 0; c < nchunks; ++c, ++gc) {
        const int buf = gc & 1;
        mbar_wait(acc_full + buf, (gc >> 1) & 1);
        tc_fence_after();
        argmax_chunk<BIAS>(tmem + lane_off + (buf * TILES + t) * 128, nch, c * nch, ks, bias_row, best, best_j, keep);
        tc_fence_before();
        mbar_arrive(acc_empty + buf);
      }
      best_j = argmax_finish(best, best_j, keep);
      const int n = n0 + t * BM + r;
      if (n < N) labels[(size_t)bh * N + n] = best_j;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == WARP_MMA) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ---------------------------------------------------------------------------------------------
// One-chunk form (ks <= 128, the query side) with hi and lo concatenated along N instead of K: the
// B operand of a K = 16 step is the 2 nch rows [W_hi ; W_lo] (two TMA boxes of the same Wsplit rows,
// columns s 64.. and D + s 64..), so each token tile takes D / 16 MMAs of N = 2 nch instead of 2 D / 16
// of N = nch: the X tile is read from shared memory once per K-step instead of twice, and the
// instructions are wide enough to reach the tensor floor (an SS instruction at N <= 128 costs
// ~80 cycles whatever N is, scripts/micro/mma_shapes.cu).  score_j = acc[j] + acc[nch + j] (+ bias),
// then the same grouped argmax.  TMEM: one 2 nch <= 256-column accumulator per token tile (the two
// tiles of a unit: tile 0's epilogue overlaps tile 1's MMAs and tile 1's the next unit's tile 0).
// W (2 slabs of 2 nch x 64 columns) stays resident across a head's units.
// ---------------------------------------------------------------------------------------------
template <int D>
struct SmemNC {
  static constexpr int HALVES = D / 64;
  static constexpr int XT = BM * D * 2;
  static constexpr int HALF_X = BM * 128;
  static constexpr int XSTAGE = TILES * XT;
  static constexpr int SLAB = 2 * NCH_MAX * 128;  // 64 columns x (hi rows ; lo rows)
  static constexpr int OFF_X = 0;
  static constexpr int OFF_W = OFF_X + 2 * XSTAGE;
  static constexpr int OFF_BAR = OFF_W + HALVES * SLAB;
  // x_full[2], x_empty[2], w_full[HALVES], w_empty[HALVES], acc_full[2], acc_empty[2]
  static constexpr int OFF_MISC = OFF_BAR + 8 * 16;
  static constexpr int BYTES = OFF_MISC + 16;
  static constexpr int ALLOC = BYTES + 1024;
};

template <int D, bool BIAS>
__global__ void __launch_bounds__(NTHREADS, 1)
    k_assign_nc(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_w,
                int H, int N, int ks, int nch, int ks_pad, int units_per_head, int num_units,
                const float* __restrict__ bias, int32_t* __restrict__ labels) {
  using L = SmemNC<D>;
  constexpr int SLABS = L::HALVES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L::OFF_BAR);
  uint64_t* x_full = bars;
  uint64_t* x_empty = bars + 2;
  uint64_t* w_full = bars + 4;
  uint64_t* w_empty = bars + 4 + SLABS;
  uint64_t* acc_full = bars + 4 + 2 * SLABS;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + L::OFF_MISC);

  const int warp = warp_id(), lane = lane_id();
  const int upc = (num_units + gridDim.x - 1) / gridDim.x;
  const int u_begin = blockIdx.x * upc, u_end = min(num_units, u_begin + upc);
  const int slab_bytes = 2 * nch * 128;

  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) { mbar_init(x_full + s, 1); mbar_init(x_empty + s, 1); }
    for (int s = 0; s < SLABS; ++s) { mbar_init(w_full + s, 1); mbar_init(w_empty + s, 1); }
    for (int t = 0; t < 2; ++t) { mbar_init(acc_full + t, 1); mbar_init(acc_empty + t, BM); }
    fence_barrier_init();
  }
  if (warp == WARP_MMA) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == WARP_PRODUCER) {
    if (lane == 0) {
      tma_prefetch_desc(&tm_x);
      tma_prefetch_desc(&tm_w);
      int it = 0, prev_bh = -1;
      for (int u = u_begin; u < u_end; ++u, ++it) {
        const int bh = u / units_per_head, n0 = (u % units_per_head) * (TILES * BM);
        const int b = bh / H, h = bh % H;
        const int xs = it & 1;
        mbar_wait(x_empty + xs, ((it >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(x_full + xs, L::XSTAGE);
        for (int t = 0; t < TILES; ++t)
          for (int hf = 0; hf < L::HALVES; ++hf)
            tma_load_4d(sm + L::OFF_X + xs * L::XSTAGE + t * L::XT + hf * L::HALF_X, &tm_x, hf * 64,
                        n0 + t * BM, h, b, x_full + xs);
        for (int s = 0; s < SLABS; ++s) {
          mbar_wait(w_empty + s, (it & 1) ^ 1);
          if (bh == prev_bh) {
            mbar_arrive(w_full + s);  // same head: the slab is still resident
          } else {
            mbar_arrive_expect_tx(w_full + s, slab_bytes);
            uint8_t* dst = sm + L::OFF_W + s * L::SLAB;
            tma_load_2d(dst, &tm_w, s * 64, bh * ks_pad, w_full + s);                  // W_hi rows
            tma_load_2d(dst + nch * 128, &tm_w, D + s * 64, bh * ks_pad, w_full + s);  // W_lo rows
          }
        }
        prev_bh = bh;
      }
    }
  } else if (warp == WARP_MMA) {
    if (lane == 0) {
      const uint32_t idesc = idesc_bf16(BM, 2 * nch, 0, 0);
      const uint32_t sX = smem_u32(sm + L::OFF_X), sW = smem_u32(sm + L::OFF_W);
      int it = 0, gt = 0;
      for (int u = u_begin; u < u_end; ++u, ++it) {
        const int xs = it & 1;
        mbar_wait(x_full + xs, (it >> 1) & 1);
        for (int s = 0; s < SLABS; ++s) mbar_wait(w_full + s, it & 1);
        tc_fence_after();
        for (int t = 0; t < TILES; ++t, ++gt) {
          mbar_wait(acc_empty + t, ((gt >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t d_tmem = tmem + t * 256;
          for (int s = 0; s < SLABS; ++s) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint64_t ad = smem_desc_sw128(sX + xs * L::XSTAGE + t * L::XT + s * L::HALF_X + k * 32, 16, 1024);
              const uint64_t bd = smem_desc_sw128(sW + s * L::SLAB + k * 32, 16, 1024);
              mma_ss(d_tmem, ad, bd, idesc, (s > 0 || k > 0) ? 1u : 0u);
            }
          }
          mma_commit(acc_full + t);
        }
        for (int s = 0; s < SLABS; ++s) mma_commit(w_empty + s);
        mma_commit(x_empty + xs);
      }
    }
    __syncwarp();
  } else {
    // epilogue: tile t = warp / 4; score_j = hi part + lo part (+ bias), grouped running argmax
    const int t = warp >> 2, quad = warp & 3;
    const int r = quad * 32 + lane;
    const uint32_t t_acc = tmem + ((uint32_t)(quad * 32) << 16) + t * 256;
    int gt = t;
    for (int u = u_begin; u < u_end; ++u, gt += TILES) {
      const int bh = u / units_per_head, n0 = (u % units_per_head) * (TILES * BM);
      float best = -INFINITY;
      int best_j = 0;
      float keep[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) keep[i] = -INFINITY;
      const float* bias_row = BIAS ? bias + (size_t)bh * ks_pad : nullptr;
      mbar_wait(acc_full + t, (gt >> 1) & 1);
      tc_fence_after();
      for (int c0 = 0; c0 < nch; c0 += 16) {
        uint32_t vh[16], vl[16];
        float bs[16];
        tmem_ld16(t_acc + c0, vh);
        tmem_ld16(t_acc + nch + c0, vl);
        if constexpr (BIAS) {
          const float4* b4 = reinterpret_cast<const float4*>(bias_row + c0);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float4 q = __ldg(b4 + i);
            bs[4 * i] = q.x; bs[4 * i + 1] = q.y; bs[4 * i + 2] = q.z; bs[4 * i + 3] = q.w;
          }
        }
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 16; ++i) vh[i] = __float_as_uint(__uint_as_float(vh[i]) + __uint_as_float(vl[i]));
        argmax_group<BIAS>(vh, bs, c0, ks, best, best_j, keep);
      }
      tc_fence_before();
      mbar_arrive(acc_empty + t);
      best_j = argmax_finish(best, best_j, keep);
      const int n = n0 + t * BM + r;
      if (n < N) labels[(size_t)bh * N + n] = best_j;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == WARP_MMA) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

}  // namespace asg

// ---------------------------------------------------------------------------------------------
// CTA-pair variant (cta_group::2) for centroid sides of more than one chunk (the key side, K_k >
// 128).  A cluster of 2 CTAs (one per SM of a TPC) owns a unit of 256 tokens: CTA r holds token
// tile r (rows n0 + 128 r ...), and each 64-column W slab of an N <= 256 chunk is split by rows
// between the two CTAs (CTA r loads chunk rows [r nch/2, (r+1) nch/2)).  The leader issues M=256
// MMAs; each CTA's TMEM receives its own 128 token rows x nch columns.  Per SM this reads 4 KB of
// A and nch/2 x 32 B of B per K=16 step and receives half of the streamed W (shared-
// memory budget), and when the head's whole W fits the 8-slab ring (nchunks x slabs = 8, e.g.
// K_k = 500 -> 2 chunks of 256) it stays resident across the head's units, so W is not re-streamed.
// Warps 0-3: epilogue (thread = token row), warp 4: TMA producer, warp 5: TMEM allocator + MMA
// issuer (leader only).
namespace asg2 {
constexpr int BM = 128, NTHREADS = 192, NCH_MAX = 256;
constexpr int WARP_PRODUCER = 4, WARP_MMA = 5;

// XST token-tile stages, NSTW W-slab stages; launched as (2, 8): the whole W of a head fits the
// ring at K_k <= 512 (2 chunks x 4 slabs at d = 128)
template <int D, int XST, int NSTW>
struct Smem {
  static constexpr int HALVES = D / 64;
  static constexpr int XT = BM * D * 2;             // this CTA's 128-token tile
  static constexpr int HALF_X = BM * 128;
  static constexpr int SLAB = (NCH_MAX / 2) * 128;  // this CTA's half of a 64-column W slab
  static constexpr int OFF_X = 0;
  static constexpr int OFF_W = OFF_X + XST * XT;
  static constexpr int OFF_BAR = OFF_W + NSTW * SLAB;
  // x_full[XST], x_empty[XST], w_full[NSTW], w_empty[NSTW], acc_full[2], acc_empty[2]
  static constexpr int OFF_MISC = OFF_BAR + (2 * XST + 2 * NSTW + 4) * 8;
  static constexpr int BYTES = OFF_MISC + 16;
  static constexpr int ALLOC = BYTES + 1024;
};

template <int D, bool BIAS, int XST, int NSTW>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NTHREADS, 1)
    k_assign_pair(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_w,
                  int H, int N, int ks, int nch, int ks_pad, int units_per_head, int num_units,
                  const float* __restrict__ bias, int32_t* __restrict__ labels) {
  using L = Smem<D, XST, NSTW>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L::OFF_BAR);
  uint64_t* x_full = bars;
  uint64_t* x_empty = bars + XST;
  uint64_t* w_full = bars + 2 * XST;
  uint64_t* w_empty = w_full + NSTW;
  uint64_t* acc_full = w_empty + NSTW;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + L::OFF_MISC);

  const int warp = warp_id(), lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const int nchunks = ks_pad / nch;
  const int half = nch / 2;
  const int ncl = gridDim.x / 2, cid = blockIdx.x / 2;
  const int upc = (num_units + ncl - 1) / ncl;
  const int u_begin = cid * upc, u_end = min(num_units, u_begin + upc);
  constexpr int SLABS = 2 * D / 64;
  const bool can_reside = nchunks * SLABS == NSTW;

  if (threadIdx.x == 0) {
    for (int s = 0; s < XST; ++s) { mbar_init(x_full + s, 1); mbar_init(x_empty + s, 1); }
    for (int s = 0; s < NSTW; ++s) { mbar_init(w_full + s, 1); mbar_init(w_empty + s, 1); }
    for (int t = 0; t < 2; ++t) { mbar_init(acc_full + t, 1); mbar_init(acc_empty + t, 8); }
    fence_barrier_init();
  }
  // Both CTAs past their prologue before the collective CTA-pair alloc: without this barrier
  // compute-sanitizer racecheck reports the peer's half of tcgen05.alloc.cta_group::2 writing
  // the slot while this CTA's alloc accesses it (scripts/micro/pair_alloc_race.cu: variants 2/3
  // report it, variant 4 = this barrier does not; once per persistent CTA).
  cluster_sync_all();
  if (warp == WARP_MMA) tmem_alloc_pair(tmem_slot, 512);
  tc_fence_before();
  cluster_sync_all();  // barriers initialised and TMEM allocated in both CTAs
  __syncthreads();     // (also a CTA barrier, which compute-sanitizer's racecheck models)
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == WARP_PRODUCER) {
    if (lane == 0) {
      tma_prefetch_desc(&tm_x);
      tma_prefetch_desc(&tm_w);
      int g = 0, it = 0, prev_bh = -1;
      for (int u = u_begin; u < u_end; ++u, ++it) {
        const int bh = u / units_per_head, n0 = (u % units_per_head) * (2 * BM);
        const int b = bh / H, h = bh % H;
        const int xs = it % XST;
        mbar_wait(x_empty + xs, ((it / XST) & 1) ^ 1);
        const uint32_t xf = mapa_shared(smem_u32(x_full + xs), 0);
        if (rank == 0) mbar_arrive_expect_tx(x_full + xs, 2 * L::XT);
        for (int hf = 0; hf < L::HALVES; ++hf)
          tma_load_4d_pair(sm + L::OFF_X + xs * L::XT + hf * L::HALF_X, &tm_x, hf * 64, n0 + (int)rank * BM, h, b,
                           xf);
        const bool resident = can_reside && bh == prev_bh;
        for (int c = 0; c < nchunks; ++c)
          for (int s = 0; s < SLABS; ++s, ++g) {
            const int stage = g % NSTW;
            mbar_wait(w_empty + stage, ((g / NSTW) & 1) ^ 1);
            if (resident) {
              if (rank == 0) mbar_arrive(w_full + stage);
            } else {
              if (rank == 0) mbar_arrive_expect_tx(w_full + stage, nch * 128);
              tma_load_2d_pair(sm + L::OFF_W + stage * L::SLAB, &tm_w, s * 64, bh * ks_pad + c * nch + (int)rank * half,
                               mapa_shared(smem_u32(w_full + stage), 0));
            }
          }
        prev_bh = bh;
      }
    }
  } else if (warp == WARP_MMA) {
    if (lane == 0 && rank == 0) {
      const uint32_t idesc = idesc_bf16(2 * BM, nch, 0, 0);
      const uint32_t sX = smem_u32(sm + L::OFF_X), sW = smem_u32(sm + L::OFF_W);
      int g = 0, gc = 0, it = 0;
      for (int u = u_begin; u < u_end; ++u, ++it) {
        const int xs = it % XST;
        mbar_wait(x_full + xs, (it / XST) & 1);
        for (int c = 0; c < nchunks; ++c, ++gc) {
          const int buf = gc & 1;
          mbar_wait(acc_empty + buf, ((gc >> 1) & 1) ^ 1);
          tc_fence_after();
          for (int s = 0; s < SLABS; ++s, ++g) {
            const int stage = g % NSTW;
            mbar_wait(w_full + stage, (g / NSTW) & 1);
            tc_fence_after();
            const int xh = s % L::HALVES;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint64_t ad = smem_desc_sw128(sX + xs * L::XT + xh * L::HALF_X + k * 32, 16, 1024);
              const uint64_t bd = smem_desc_sw128(sW + stage * L::SLAB + k * 32, 16, 1024);
              mma_ss_pair(tmem + buf * NCH_MAX, ad, bd, idesc, (s > 0 || k > 0) ? 1u : 0u);
            }
            mma_commit_pair(w_empty + stage);
          }
          mma_commit_pair(acc_full + buf);
        }
        mma_commit_pair(x_empty + xs);
      }
    }
    __syncwarp();
  } else {
    // epilogue: grouped running argmax (as k_assign), ties -> lowest index
    const int r = warp * 32 + lane;
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    int gc = 0;
    for (int u = u_begin; u < u_end; ++u) {
      const int bh = u / units_per_head, n0 = (u % units_per_head) * (2 * BM);
      float best = -INFINITY;
      int best_j = 0;
      float keep[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) keep[i] = -INFINITY;
      const float* bias_row = BIAS ? bias + (size_t)bh * ks_pad : nullptr;
      for (int c = 0; c < nchunks; ++c, ++gc) {
        const int buf = gc & 1;
        mbar_wait(acc_full + buf, (gc >> 1) & 1);
        tc_fence_after();
        asg::argmax_chunk<BIAS>(tmem + lane_off + buf * NCH_MAX, nch, c * nch, ks, bias_row, best, best_j, keep);
        tc_fence_before();
        __syncwarp();
        // relaxed: the TMEM reads are complete (tcgen05.wait::ld), nothing in memory to publish; a
        // release arrive at cluster scope costs a memory barrier per chunk (ncu: ERRBAR, 13 % of
        // the kernel's stall samples)
        if (lane == 0) {
#ifdef CS_ARRIVE_RELEASE
          mbar_arrive_cluster(mapa_shared(smem_u32(acc_empty + buf), 0));
#else
          mbar_arrive_cluster_relaxed(mapa_shared(smem_u32(acc_empty + buf), 0));
#endif
        }
      }
      best_j = asg::argmax_finish(best, best_j, keep);
      const int n = n0 + (int)rank * BM + r;
      if (n < N) labels[(size_t)bh * N + n] = best_j;
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == WARP_MMA) {
    tc_fence_after();
    tmem_dealloc_pair(tmem, 512);
  }
}
}  // namespace asg2

#ifndef CS_ASSIGN_PAIR
#define CS_ASSIGN_PAIR 1
#endif
// ks <= 128 (one chunk, e.g. the query side): single-CTA kernel, N = ks rounded to 16, W resident
// across a head's units (the pair kernel with 4 token stages measured slower there: 233 vs 186 us
// at K_q = 100, an HBM-bound launch).  More: the CTA-pair kernel with ceil(ks / 256) chunks of
// N <= 256 (a multiple of 32, so each CTA holds a multiple of 16 rows).  CS_ASSIGN_PAIR=0 builds
// the single-CTA kernel for every side (A/B comparisons).
static bool use_pair(int ks) { return CS_ASSIGN_PAIR && ks > asg::NCH_MAX; }
int assign_chunk_n(int ks) {
  if (!use_pair(ks)) return ks <= asg::NCH_MAX ? (ks + 15) / 16 * 16 : asg::NCH_MAX;
  const int nchunks = (ks + asg2::NCH_MAX - 1) / asg2::NCH_MAX;
  return ((ks + nchunks - 1) / nchunks + 31) / 32 * 32;
}
int assign_box_rows(int ks) { return use_pair(ks) ? assign_chunk_n(ks) / 2 : assign_chunk_n(ks); }

cudaError_t launch_assign_gemm(const CUtensorMap* tm_x, const CUtensorMap* tm_w, int B, int H, int N,
                               int d, int ks, int nch, int ks_pad, const float* bias, int32_t* labels,
                               cudaStream_t st) {
  int num_sms = 0, dev = 0;  // queried per call: no shared mutable state, right for any current device
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
  if (num_sms <= 0) num_sms = 148;
  const int units_per_head = (N + asg::TILES * asg::BM - 1) / (asg::TILES * asg::BM);
  const int num_units = units_per_head * B * H;
  if (use_pair(ks)) {
    const int pairs = num_units < num_sms / 2 ? num_units : num_sms / 2;
    auto launch2 = [&](auto kfn, int smem) -> cudaError_t {
      cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (e != cudaSuccess) return e;
      kfn<<<2 * pairs, asg2::NTHREADS, smem, st>>>(*tm_x, *tm_w, H, N, ks, nch, ks_pad, units_per_head, num_units,
                                                    bias, labels);
      return cudaSuccess;
    };
    cudaError_t e;
    using namespace asg2;
    if (d == 128)
      e = bias ? launch2(k_assign_pair<128, true, 2, 8>, Smem<128, 2, 8>::ALLOC)
               : launch2(k_assign_pair<128, false, 2, 8>, Smem<128, 2, 8>::ALLOC);
    else
      e = bias ? launch2(k_assign_pair<64, true, 2, 8>, Smem<64, 2, 8>::ALLOC)
               : launch2(k_assign_pair<64, false, 2, 8>, Smem<64, 2, 8>::ALLOC);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
  }
  const int grid = num_units < num_sms ? num_units : num_sms;
#ifndef CS_ASSIGN_NC
#define CS_ASSIGN_NC 1
#endif
  if (CS_ASSIGN_NC && ks_pad == nch && 2 * nch <= 256) {
    auto launch_nc = [&](auto kfn, int smem) -> cudaError_t {
      cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (e != cudaSuccess) return e;
      kfn<<<grid, asg::NTHREADS, smem, st>>>(*tm_x, *tm_w, H, N, ks, nch, ks_pad, units_per_head, num_units, bias,
                                             labels);
      return cudaSuccess;
    };
    cudaError_t e;
    if (d == 128)
      e = bias ? launch_nc(asg::k_assign_nc<128, true>, asg::SmemNC<128>::ALLOC)
               : launch_nc(asg::k_assign_nc<128, false>, asg::SmemNC<128>::ALLOC);
    else
      e = bias ? launch_nc(asg::k_assign_nc<64, true>, asg::SmemNC<64>::ALLOC)
               : launch_nc(asg::k_assign_nc<64, false>, asg::SmemNC<64>::ALLOC);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
  }
  auto launch = [&](auto kfn, int smem) -> cudaError_t {
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    kfn<<<grid, asg::NTHREADS, smem, st>>>(*tm_x, *tm_w, H, N, ks, nch, ks_pad, units_per_head, num_units, bias,
                                           labels);
    return cudaSuccess;
  };
  cudaError_t e;
  if (d == 128)
    e = bias ? launch(asg::k_assign<128, true>, asg::Smem<128>::ALLOC) : launch(asg::k_assign<128, false>, asg::Smem<128>::ALLOC);
  else
    e = bias ? launch(asg::k_assign<64, true>, asg::Smem<64>::ALLOC) : launch(asg::k_assign<64, false>, asg::Smem<64>::ALLOC);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace cs
