// profile.cu — offline layer-wise sparsity profiling on sm_100a.
//
// Attention density of one head: d = (1/N) sum_i |S(i)| / N, where S(i) is the minimal descending
// prefix of row i of A = softmax(q k^T * scale) whose mass reaches tau (R9b tolerance 1e-12).
// A full per-row sort over N = 75,600 columns is replaced by a radix select on the float bits of
// the unnormalised probabilities p_ij = 2^(s_ij * scale * log2(e) - m_i) in (0, 1] (positive
// floats order like their bit patterns):
//   pass 0      : row max m_i and Z_i = sum_j p_ij                          (online, like flash)
//   pass 1      : 32 bins by the exponent of p (2^-32 < p <= 1; smaller p carry < 1e-4 of the mass
//                 at N <= 2^17, so the tau crossing is never below them); every element adds p and
//                 1 to its bin, the bin where the descending cumulative mass crosses tau Z_i
//                 becomes the prefix of the next pass, the bins above it are carried (mass, count)
//   pass k >= 2 : 32 bins by the next 5 mantissa bits among the elements matching the prefix
//                 (one AND/XOR and a min per element; a 32-column chunk of a thread without a
//                 match skips the binning)
//   the last pass converts the crossing bin (p known to 5 (P-1) mantissa bits) into a count:
//   elements above + ceil(residual mass / mean mass of the bin's elements).
// Each pass recomputes S = Q K^T with tcgen05 (QK only: no PV, no P): one CTA = two 128-row Q
// tiles of one head against every 128-key tile (2-slot TMA ring, TMEM double-buffered S for both
// tiles), 8 row-worker warps (thread = query row = TMEM lane) + 1 TMA producer + 1 MMA warp.
// Per-row bins live in shared memory as [bin][row] (one thread per row: conflict-free, no atomics).
#include "kernels.cuh"

namespace cs {
namespace dens {

constexpr int BM = 128, BN = 128, NST = 2, NBIN = 32, NTHREADS = 320;
constexpr int WARP_PRODUCER = 8, WARP_MMA = 9;

template <int D>
struct Smem {
  static constexpr int HALVES = D / 64;
  static constexpr int QT = BM * D * 2, KT = BN * D * 2;
  static constexpr int HALF_Q = BM * 128, HALF_K = BN * 128;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + 2 * QT;
  static constexpr int OFF_BINS = OFF_K + NST * KT;              // float2 {mass, count bits} [NBIN][2 BM]
  static constexpr int OFF_BAR = OFF_BINS + NBIN * 2 * BM * 8;   // q_full, k_full[2], k_empty[2], s_full[2], s_empty[2]
  static constexpr int OFF_MISC = OFF_BAR + 16 * 8;
  static constexpr int BYTES = OFF_MISC + 16;
  static constexpr int ALLOC = BYTES + 1024;
};

// pass 0 stats: m = max_j s_ij * c (c = scale log2 e), z = sum_j 2^(s_ij c - m)
// pass p >= 1: bins over [lo, hi); last pass writes counts
template <int D>
__global__ void __launch_bounds__(NTHREADS, 1)
    k_density(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k, int H, int N,
              float c, int pass, int last, double tau, float* __restrict__ rs, size_t rows,
              int32_t* __restrict__ counts) {
  // per-row state [6][rows]: m, Z, lo, hi, mass above hi, count above hi (int bits)
  float* row_m = rs;
  float* row_z = rs + rows;
  float* row_lo = rs + 2 * rows;
  float* row_hi = rs + 3 * rows;
  float* row_am = rs + 4 * rows;
  int* row_an = reinterpret_cast<int*>(rs + 5 * rows);
  using L = Smem<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L::OFF_BAR);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;
  uint64_t* k_empty = bars + 3;
  uint64_t* s_full = bars + 5;
  uint64_t* s_empty = bars + 7;
  uint2* bins = reinterpret_cast<uint2*>(sm + L::OFF_BINS);  // .x = mass (fp32 bits), .y = count
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
    float m = -INFINITY, z = 0.f;
    // radix state: elements with (bits(p) & pmask) == prefix are binned by (bits(p) >> sh) & 31
    // (pass 1: the exponent, bins 0..31 = exponents 96..127)
    uint32_t prefix = 0u, pmask = 0u;
    const int sh = pass <= 1 ? 23 : 18 - 5 * (pass - 2);
    if (pass > 0) {
      m = row_ok ? row_m[ridx] : 0.f;
      if (pass > 1) {
        prefix = row_ok ? __float_as_uint(row_lo[ridx]) : 0xffffffffu;
        pmask = 0xffffffffu << (sh + 5);
      }
#pragma unroll
      for (int bi = 0; bi < NBIN; ++bi) bins[bi * 2 * BM + col] = make_uint2(0u, 0u);
    }
    float above = 0.f;  // mass / count of the elements above the current prefix (carried)
    int above_n = 0;
    if (pass > 1 && row_ok) { above = row_am[ridx]; above_n = row_an[ridx]; }
    auto bin_of = [&](uint32_t u) -> int {  // -1: not binned in this pass
      if (pass == 1) {
        const int e = (int)(u >> 23) - 96;
        return e >= 0 ? min(e, NBIN - 1) : -1;
      }
      return (u & pmask) == prefix ? (int)((u >> sh) & 31u) : -1;
    };
    for (int j = 0; j < nt; ++j) {
      const int buf = j & 1;
      mbar_wait(s_full + buf, (j >> 1) & 1);
      tc_fence_after();
      const uint32_t s_tm = tmem + lane_off + (buf * 2 + t) * 128;
      const int valid = min(BN, N - j * BN);  // columns past N (TMA zero fill) are ignored
      float mx = -INFINITY;
      if (pass == 0) {  // the row max of this tile first (a second TMEM read below)
#pragma unroll 1
        for (int cc = 0; cc < BN / 32; ++cc) {
          uint32_t su[32];
          tmem_ld32(s_tm + cc * 32, su);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) mx = fmaxf(mx, cc * 32 + i < valid ? __uint_as_float(su[i]) : -INFINITY);
        }
        const float mn = fmaxf(m, mx * c);
        z *= ex2(m - mn);  // m = -inf on the first tile: ex2(-inf) = 0
        m = mn;
      }
#pragma unroll 1
      for (int cc = 0; cc < BN / 32; ++cc) {
        uint32_t su[32];
        tmem_ld32(s_tm + cc * 32, su);
        tmem_wait_ld();
        if (cc == BN / 32 - 1) {  // the S buffer is free for the MMA of tile j + 2
          tc_fence_before();
          mbar_arrive(s_empty + buf);
        }
        const bool tail = cc * 32 + 32 > valid;  // warp-uniform: only the last key tile has a tail
        if (pass == 0) {
          float acc = 0.f;
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float e = ex2(fmaf(__uint_as_float(su[i]), c, -m));
            acc += (!tail || cc * 32 + i < valid) ? e : 0.f;
          }
          z += acc;
          continue;
        }
        // p = 2^x as bits; columns past N -> 0 (never binned: exponent 0)
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const uint32_t u = __float_as_uint(ex2(fmaf(__uint_as_float(su[i]), c, -m)));
          su[i] = (!tail || cc * 32 + i < valid) ? u : 0u;
        }
        if (pass > 1) {
          // narrow prefix: few matches per row -> visit only those
          uint32_t mn2 = 0xffffffffu;
#pragma unroll
          for (int i = 0; i < 32; ++i) mn2 = min(mn2, (su[i] & pmask) ^ prefix);
          if (mn2 != 0u) continue;  // no element of this thread's chunk matches
          uint32_t inm = 0u;
#pragma unroll
          for (int i = 0; i < 32; ++i) inm |= ((su[i] & pmask) == prefix) ? (1u << i) : 0u;
          while (inm) {
            const int i = __ffs(inm) - 1;
            inm &= inm - 1;
            uint32_t ui = su[0];
#pragma unroll
            for (int k2 = 1; k2 < 32; ++k2) ui = k2 == i ? su[k2] : ui;  // register select, no local memory
            const int b = (int)((ui >> sh) & 31u);
            const uint2 v = bins[b * 2 * BM + col];
            bins[b * 2 * BM + col] = make_uint2(__float_as_uint(__uint_as_float(v.x) + __uint_as_float(ui)), v.y + 1u);
          }
          continue;
        }
        // pass 1 (every element): groups of G; duplicate bins inside a group are merged first, so
        // the G read-modify-writes of a group hit distinct SMEM words and issue back to back
        constexpr int G = 4;
#pragma unroll
        for (int i0 = 0; i0 < 32; i0 += G) {
          int bk[G], cn[G];
          float pm[G];
#pragma unroll
          for (int g = 0; g < G; ++g) {
            const int b = bin_of(su[i0 + g]);
            bk[g] = b >= 0 ? b : -1 - g;  // unique negative: no bin
            pm[g] = b >= 0 ? __uint_as_float(su[i0 + g]) : 0.f;
            cn[g] = b >= 0 ? 1 : 0;
          }
#pragma unroll
          for (int g = 1; g < G; ++g)
#pragma unroll
            for (int h2 = 0; h2 < g; ++h2)
              if (bk[h2] == bk[g]) {  // bk[h2] is the first occurrence (merged ones get -8 - g)
                pm[h2] += pm[g];
                cn[h2] += cn[g];
                bk[g] = -8 - g;
              }
          uint2 v[G];
#pragma unroll
          for (int g = 0; g < G; ++g)
            if (bk[g] >= 0) v[g] = bins[bk[g] * 2 * BM + col];
#pragma unroll
          for (int g = 0; g < G; ++g)
            if (bk[g] >= 0)
              bins[bk[g] * 2 * BM + col] = make_uint2(__float_as_uint(__uint_as_float(v[g].x) + pm[g]), v[g].y + cn[g]);
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
          const uint2 bv = bins[bi * 2 * BM + col];
          const float bm = __uint_as_float(bv.x);
          if (cum + bm >= T) { cb = bi; break; }
          cum += bm;
          cnt += (int)bv.y;
        }
        if (!last) {
          const int bsel = cb < 0 ? 0 : cb;
          const uint32_t np = pass == 1 ? (uint32_t)(96 + bsel) << 23 : prefix | ((uint32_t)bsel << sh);
          row_lo[ridx] = __uint_as_float(np);  // the next pass's prefix (bits)
          row_am[ridx] = cum;  // mass / count of the bins above the chosen one (and above hi)
          row_an[ridx] = cnt;
        } else {
          int need = 0;
          if (cb >= 0 && cum < T) {
            const uint2 bv = bins[cb * 2 * BM + col];
            const int bn_ = (int)bv.y;
            const float mean = __uint_as_float(bv.x) / (float)max(bn_, 1);
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
                                     float scale, double tau, int passes, float* rs, size_t rows, int32_t* counts,
                                     double* density, cudaStream_t st) {
  const float c = scale * 1.4426950408889634f;
  const dim3 grid((N + 2 * dens::BM - 1) / (2 * dens::BM), B * H);
  auto run = [&](auto kfn, int smem) -> cudaError_t {
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    for (int p = 0; p <= passes; ++p)
      kfn<<<grid, dens::NTHREADS, smem, st>>>(*tm_q, *tm_k, H, N, c, p, p == passes ? 1 : 0, tau, rs, rows,
                                             counts);
    return cudaGetLastError();
  };
  cudaError_t e = d == 128 ? run(dens::k_density<128>, dens::Smem<128>::ALLOC)
                           : run(dens::k_density<64>, dens::Smem<64>::ALLOC);
  if (e != cudaSuccess) return e;
  dens::k_density_reduce<<<B * H, 1024, 0, st>>>(N, counts, density);
  return cudaGetLastError();
}

}  // namespace cs
