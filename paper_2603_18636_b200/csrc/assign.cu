// assign.cu — Alg. 1 assignment (Step A: P:1214-1218, Step B: P:1222-1226) as a tcgen05 GEMM with
// a fused row-argmax epilogue, in the exact reduced form:
//     L(i) = argmin_j || Norm(x_i C_a^T) - Norm(c_j C_a^T) ||_2 = argmax_j x_i . W_j,
//     W_j  = (C_a^T C_a) c_j / ||c_j C_a^T||   (ties -> lowest j)
// W enters the tensor core as two bf16 parts (hi + lo), so each score is
//     x_i . W_hi_j + x_i . W_lo_j   accumulated in fp32 over an inner dimension of 2d.
//
// One CTA = 128 tokens of one head (M = 128).  The centroid side is streamed in chunks of
// nch <= 256 columns (UMMA N = nch) through a 4-stage ring of 64-column W slabs; the fp32 score
// tile lives in TMEM (2 buffers x nch columns) so the argmax epilogue of chunk c overlaps the
// MMAs of chunk c+1.  Warps 0-3: epilogue (thread = token row = TMEM lane), warp 4: TMA producer,
// warp 5: TMEM allocator + MMA issuer.
#include "kernels.cuh"

namespace cs {
namespace asg {

constexpr int BM = 128, NSTW = 4, NTHREADS = 192;
constexpr int WARP_PRODUCER = 4, WARP_MMA = 5;

template <int D>
struct Smem {
  static constexpr int HALVES = D / 64;
  static constexpr int XT = BM * D * 2;
  static constexpr int HALF_X = BM * 128;
  static constexpr int SLAB = 256 * 128;  // max nch rows x 128 B
  static constexpr int OFF_X = 0;
  static constexpr int OFF_W = OFF_X + XT;
  static constexpr int OFF_BAR = OFF_W + NSTW * SLAB;
  // x_full, w_full[4], w_empty[4], acc_full[2], acc_empty[2]
  static constexpr int OFF_MISC = OFF_BAR + 8 * 16;
  static constexpr int BYTES = OFF_MISC + 16;
  static constexpr int ALLOC = BYTES + 1024;
};

template <int D>
__global__ void __launch_bounds__(NTHREADS, 1)
    k_assign(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_w,
             int H, int N, int ks, int nch, int ks_pad, int32_t* __restrict__ labels) {
  using L = Smem<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L::OFF_BAR);
  uint64_t* x_full = bars;
  uint64_t* w_full = bars + 1;
  uint64_t* w_empty = bars + 1 + NSTW;
  uint64_t* acc_full = bars + 1 + 2 * NSTW;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + L::OFF_MISC);

  const int bh = blockIdx.y, b = bh / H, h = bh % H;
  const int n0 = blockIdx.x * BM;
  const int warp = warp_id(), lane = lane_id();
  const int nchunks = ks_pad / nch;
  constexpr int SLABS = 2 * D / 64;  // 64-column slabs per chunk (hi halves then lo halves)
  const int total_slabs = nchunks * SLABS;

  if (threadIdx.x == 0) {
    mbar_init(x_full, 1);
    for (int s = 0; s < NSTW; ++s) { mbar_init(w_full + s, 1); mbar_init(w_empty + s, 1); }
    for (int t = 0; t < 2; ++t) { mbar_init(acc_full + t, 1); mbar_init(acc_empty + t, 128); }
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
      mbar_arrive_expect_tx(x_full, L::XT);
      for (int hf = 0; hf < L::HALVES; ++hf)
        tma_load_4d(sm + L::OFF_X + hf * L::HALF_X, &tm_x, hf * 64, n0, h, b, x_full);
      for (int g = 0; g < total_slabs; ++g) {
        const int stage = g % NSTW;
        mbar_wait(w_empty + stage, ((g / NSTW) & 1) ^ 1);
        const int c = g / SLABS, s = g % SLABS;
        mbar_arrive_expect_tx(w_full + stage, nch * 128);
        tma_load_2d(sm + L::OFF_W + stage * L::SLAB, &tm_w, s * 64, bh * ks_pad + c * nch, w_full + stage);
      }
    }
  } else if (warp == WARP_MMA) {
    if (lane == 0) {
      const uint32_t idesc = idesc_bf16(BM, nch, 0, 0);  // N varies at run time
      const uint32_t sX = smem_u32(sm + L::OFF_X), sW = smem_u32(sm + L::OFF_W);
      mbar_wait(x_full, 0);
      for (int c = 0; c < nchunks; ++c) {
        const int buf = c & 1;
        mbar_wait(acc_empty + buf, ((c >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem + buf * 256;
        for (int s = 0; s < SLABS; ++s) {
          const int g = c * SLABS + s, stage = g % NSTW;
          mbar_wait(w_full + stage, (g / NSTW) & 1);
          tc_fence_after();
          const int xh = s % L::HALVES;  // slab s pairs with x half (s mod halves)
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint64_t ad = smem_desc_sw128(sX + xh * L::HALF_X + k * 32, 16, 1024);
            const uint64_t bd = smem_desc_sw128(sW + stage * L::SLAB + k * 32, 16, 1024);
            mma_ss(d_tmem, ad, bd, idesc, (s > 0 || k > 0) ? 1u : 0u);
          }
          mma_commit(w_empty + stage);
        }
        mma_commit(acc_full + buf);
      }
    }
    __syncwarp();
  } else {
    // epilogue: running argmax over the valid centroid columns, ties -> lowest index
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    float best = -INFINITY;
    int best_j = 0;
    for (int c = 0; c < nchunks; ++c) {
      const int buf = c & 1;
      mbar_wait(acc_full + buf, (c >> 1) & 1);
      tc_fence_after();
      const uint32_t t_acc = tmem + lane_off + buf * 256;
      const int jbase = c * nch;
      for (int c0 = 0; c0 < nch; c0 += 16) {
        uint32_t v[16];
        tmem_ld16(t_acc + c0, v);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int j = jbase + c0 + i;
          const float x = __uint_as_float(v[i]);
          if (j < ks && x > best) { best = x; best_j = j; }
        }
      }
      tc_fence_before();
      mbar_arrive(acc_empty + buf);
    }
    if (n0 + r < N) labels[(size_t)bh * N + n0 + r] = best_j;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == WARP_MMA) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

}  // namespace asg

cudaError_t launch_assign_gemm(const CUtensorMap* tm_x, const CUtensorMap* tm_w, int B, int H, int N,
                               int d, int ks, int nch, int ks_pad, int32_t* labels, cudaStream_t st) {
  dim3 grid((N + asg::BM - 1) / asg::BM, B * H);
  if (d == 128) {
    auto kfn = asg::k_assign<128>;
    const int smem = asg::Smem<128>::ALLOC;
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    kfn<<<grid, asg::NTHREADS, smem, st>>>(*tm_x, *tm_w, H, N, ks, nch, ks_pad, labels);
  } else {
    auto kfn = asg::k_assign<64>;
    const int smem = asg::Smem<64>::ALLOC;
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    kfn<<<grid, asg::NTHREADS, smem, st>>>(*tm_x, *tm_w, H, N, ks, nch, ks_pad, labels);
  }
  return cudaGetLastError();
}

}  // namespace cs
