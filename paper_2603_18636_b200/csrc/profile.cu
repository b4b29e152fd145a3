// profile.cu — offline layer-wise sparsity profiling on sm_100a.
//
// Attention density of one head: d = (1/N) sum_i |S(i)| / N, where S(i) is the minimal descending
// prefix of row i of A = softmax(q k^T * scale) whose mass reaches tau (R9b tolerance 1e-12).
// A full per-row sort over N = 75,600 columns is replaced by a threshold search in the exp2
// domain (x_ij = s_ij * scale * log2(e) - m_i, p_ij = 2^x_ij / Z_i):
//   pass 0      : row max m_i and Z_i = sum_j 2^x_ij                      (online, like flash)
//   passes 1..P : the search interval [lo_i, hi_i) (initially [-64, 1)) is cut into 32 bins;
//                 every element adds 2^x to "above" (x >= hi) or to its bin (count + mass), and
//                 the bin where the descending cumulative mass crosses tau Z_i becomes the next
//                 interval (width 65 / 32^p).  The last pass converts the crossing bin into a
//                 count: elements above + ceil(residual mass / mean mass of the bin's elements).
// Each pass recomputes S = Q K^T with tcgen05 (QK only: no PV, no P): one CTA = two 128-row Q
// tiles of one head against every 128-key tile (2-slot TMA ring, TMEM double-buffered S for both
// tiles), 8 row-worker warps (thread = query row = TMEM lane) + 1 TMA producer + 1 MMA warp.
// Per-row bins live in shared memory as [bin][row] (one thread per row: conflict-free, no atomics).
#include "kernels.cuh"

namespace cs {
namespace dens {

constexpr int BM = 128, BN = 128, NST = 2, NBIN = 32, NTHREADS = 320;
constexpr int WARP_PRODUCER = 8, WARP_MMA = 9;
constexpr float kLo0 = -64.f, kHi0 = 1.f;  // initial search interval (log2 units below the row max)

template <int D>
struct Smem {
  static constexpr int HALVES = D / 64;
  static constexpr int QT = BM * D * 2, KT = BN * D * 2;
  static constexpr int HALF_Q = BM * 128, HALF_K = BN * 128;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + 2 * QT;
  static constexpr int OFF_MASS = OFF_K + NST * KT;              // float [NBIN][2 BM]
  static constexpr int OFF_CNT = OFF_MASS + NBIN * 2 * BM * 4;   // int   [NBIN][2 BM]
  static constexpr int OFF_BAR = OFF_CNT + NBIN * 2 * BM * 4;    // q_full, k_full[2], k_empty[2], s_full[2], s_empty[2]
  static constexpr int OFF_MISC = OFF_BAR + 16 * 8;
  static constexpr int BYTES = OFF_MISC + 16;
  static constexpr int ALLOC = BYTES + 1024;
};

// pass 0 stats: m = max_j s_ij * c (c = scale log2 e), z = sum_j 2^(s_ij c - m)
// pass p >= 1: bins over [lo, hi); last pass writes counts
template <int D>
__global__ void __launch_bounds__(NTHREADS, 1)
    k_density(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k, int H, int N,
              float c, int pass, int last, double tau, float* __restrict__ row_m, float* __restrict__ row_z,
              float* __restrict__ row_lo, float* __restrict__ row_hi, int32_t* __restrict__ counts) {
  using L = Smem<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L::OFF_BAR);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;
  uint64_t* k_empty = bars + 3;
  uint64_t* s_full = bars + 5;
  uint64_t* s_empty = bars + 7;
  float* bmass = reinterpret_cast<float*>(sm + L::OFF_MASS);
  int* bcnt = reinterpret_cast<int*>(sm + L::OFF_CNT);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + L::OFF_MISC);

  const int bh = blockIdx.y, b = bh / H, h = bh % H;
  const int n0 = blockIdx.x * 2 * BM;
  const bool has1 = n0 + BM < N;
  const int nt = (N + BN - 1) / BN;
  const int warp = warp_id(), lane = lane_id();

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < NST; ++s) { mbar_init(k_full + s, 1); mbar_init(k_empty + s, 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(s_full + s, 1); mbar_init(s_empty + s, 8 * 32); }
    fence_barrier_init();
  }
  if (warp == WARP_MMA) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == WARP_PRODUCER) {
    if (lane == 0) {
      tma_prefetch_desc(&tm_q);
      tma_prefetch_desc(&tm_k);
      mbar_arrive_expect_tx(q_full, (has1 ? 2 : 1) * L::QT);
      for (int t = 0; t < (has1 ? 2 : 1); ++t)
        for (int hf = 0; hf < L::HALVES; ++hf)
          tma_load_4d(sm + L::OFF_Q + t * L::QT + hf * L::HALF_Q, &tm_q, hf * 64, n0 + t * BM, h, b, q_full);
      for (int j = 0; j < nt; ++j) {
        const int slot = j % NST;
        mbar_wait(k_empty + slot, ((j / NST) & 1) ^ 1);
        mbar_arrive_expect_tx(k_full + slot, L::KT);
        for (int hf = 0; hf < L::HALVES; ++hf)
          tma_load_4d(sm + L::OFF_K + slot * L::KT + hf * L::HALF_K, &tm_k, hf * 64, j * BN, h, b, k_full + slot);
      }
    }
    __syncwarp();
  } else if (warp == WARP_MMA) {
    constexpr uint32_t idesc = idesc_bf16(BM, BN, 0, 0);
    const uint64_t dq0 = smem_desc_sw128(smem_u32(sm + L::OFF_Q), 16, 1024);
    const uint64_t dk0 = smem_desc_sw128(smem_u32(sm + L::OFF_K), 16, 1024);
    mbar_wait(q_full, 0);
    for (int j = 0; j < nt; ++j) {
      const int slot = j % NST, buf = j & 1;
      mbar_wait(s_empty + buf, ((j >> 1) & 1) ^ 1);
      mbar_wait(k_full + slot, (j / NST) & 1);
      tc_fence_after();
      if (elect_one()) {
        for (int t = 0; t < (has1 ? 2 : 1); ++t) {
          const uint32_t d_tmem = tmem + (buf * 2 + t) * 128;
          const uint64_t qd = dq0 + (uint64_t)((t * L::QT) >> 4);
          const uint64_t kd = dk0 + (uint64_t)((slot * L::KT) >> 4);
#pragma unroll
          for (int k2 = 0; k2 < D / 16; ++k2) {
            const uint32_t oq = ((k2 >> 2) * L::HALF_Q + (k2 & 3) * 32) >> 4;
            const uint32_t ok = ((k2 >> 2) * L::HALF_K + (k2 & 3) * 32) >> 4;
            mma_ss(d_tmem, qd + oq, kd + ok, idesc, k2 > 0);
          }
        }
        mma_commit(s_full + buf);
        mma_commit(k_empty + slot);
      }
      __syncwarp();
    }
  } else {
    // ================= row workers: warps 0-3 tile 0, 4-7 tile 1 =================
    const int t = warp >> 2, quad = warp & 3;
    const int r = quad * 32 + lane, col = t * BM + r;  // row of the tile, bin column in SMEM
    const int n = n0 + t * BM + r;
    const bool row_ok = n < N && (t == 0 || has1);
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const size_t ridx = (size_t)bh * N + (row_ok ? n : 0);
    float m = -INFINITY, z = 0.f, lo = kLo0, hi = kHi0, inv_w = 0.f;
    if (pass > 0) {
      m = row_ok ? row_m[ridx] : 0.f;
      if (pass > 1 && row_ok) { lo = row_lo[ridx]; hi = row_hi[ridx]; }
      inv_w = (float)NBIN / (hi - lo);
#pragma unroll
      for (int bi = 0; bi < NBIN; ++bi) { bmass[bi * 2 * BM + col] = 0.f; bcnt[bi * 2 * BM + col] = 0; }
    }
    float above = 0.f;
    int above_n = 0;
    for (int j = 0; j < nt; ++j) {
      const int buf = j & 1;
      mbar_wait(s_full + buf, (j >> 1) & 1);
      tc_fence_after();
      uint32_t su[BN];
      const uint32_t s_tm = tmem + lane_off + (buf * 2 + t) * 128;
#pragma unroll
      for (int cc = 0; cc < BN / 32; ++cc) tmem_ld32(s_tm + cc * 32, su + cc * 32);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(s_empty + buf);
      const int valid = min(BN, N - j * BN);  // columns past N (TMA zero fill) are ignored
      if (pass == 0) {
        float mx = -INFINITY;
#pragma unroll
        for (int i = 0; i < BN; ++i) mx = fmaxf(mx, i < valid ? __uint_as_float(su[i]) : -INFINITY);
        const float mn = fmaxf(m, mx * c);
        z *= ex2(m - mn);  // m = -inf on the first tile: ex2(-inf) = 0
        m = mn;
        float acc = 0.f;
#pragma unroll
        for (int i = 0; i < BN; ++i)
          acc += i < valid ? ex2(fmaf(__uint_as_float(su[i]), c, -m)) : 0.f;
        z += acc;
      } else {
#pragma unroll
        for (int i = 0; i < BN; ++i) {
          const float x = i < valid ? fmaf(__uint_as_float(su[i]), c, -m) : -INFINITY;
          if (x >= hi) {
            above += ex2(x);
            ++above_n;
          } else if (x >= lo) {
            const int bi = min(NBIN - 1, (int)((x - lo) * inv_w));
            bmass[bi * 2 * BM + col] += ex2(x);
            bcnt[bi * 2 * BM + col] += 1;
          }
        }
      }
    }
    if (row_ok) {
      if (pass == 0) {
        row_m[ridx] = m;
        row_z[ridx] = z;
      } else {
        const float T = (float)((tau - 1e-12) * (double)row_z[ridx]);
        float cum = above;
        int cnt = above_n, cb = -1;
        for (int bi = NBIN - 1; bi >= 0; --bi) {
          const float bm = bmass[bi * 2 * BM + col];
          if (cum + bm >= T) { cb = bi; break; }
          cum += bm;
          cnt += bcnt[bi * 2 * BM + col];
        }
        const float w = (hi - lo) / (float)NBIN;
        if (!last) {
          const int bsel = cb < 0 ? 0 : cb;
          row_lo[ridx] = lo + bsel * w;
          row_hi[ridx] = bsel == NBIN - 1 ? hi : lo + (bsel + 1) * w;
        } else {
          int need = 0;
          if (cb >= 0 && cum < T) {
            const int bn_ = bcnt[cb * 2 * BM + col];
            const float mean = bmass[cb * 2 * BM + col] / (float)max(bn_, 1);
            need = min(bn_, max(1, (int)ceilf((T - cum) / mean)));
          }
          counts[ridx] = max(1, cnt + need);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == WARP_MMA) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// density[bh] = sum_i counts[bh][i] / N^2 (exact integer sum)
__global__ void __launch_bounds__(1024) k_density_reduce(int N, const int32_t* __restrict__ counts,
                                                         double* __restrict__ density) {
  __shared__ long long part[32];
  const int bh = blockIdx.x;
  long long s = 0;
  for (int i = threadIdx.x; i < N; i += 1024) s += counts[(size_t)bh * N + i];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long tot = 0;
    for (int w = 0; w < 32; ++w) tot += part[w];
    density[bh] = (double)tot / (double)N / (double)N;
  }
}

}  // namespace dens

cudaError_t launch_attention_density(const CUtensorMap* tm_q, const CUtensorMap* tm_k, int B, int H, int N, int d,
                                     float scale, double tau, int passes, float* row_m, float* row_z, float* row_lo,
                                     float* row_hi, int32_t* counts, double* density, cudaStream_t st) {
  const float c = scale * 1.4426950408889634f;
  const dim3 grid((N + 2 * dens::BM - 1) / (2 * dens::BM), B * H);
  auto run = [&](auto kfn, int smem) -> cudaError_t {
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    for (int p = 0; p <= passes; ++p)
      kfn<<<grid, dens::NTHREADS, smem, st>>>(*tm_q, *tm_k, H, N, c, p, p == passes ? 1 : 0, tau, row_m, row_z,
                                             row_lo, row_hi, counts);
    return cudaGetLastError();
  };
  cudaError_t e = d == 128 ? run(dens::k_density<128>, dens::Smem<128>::ALLOC)
                           : run(dens::k_density<64>, dens::Smem<64>::ALLOC);
  if (e != cudaSuccess) return e;
  dens::k_density_reduce<<<B * H, 1024, 0, st>>>(N, counts, density);
  return cudaGetLastError();
}

}  // namespace cs
