// attn.cu — varlen block-sparse flash attention over co-clustered blocks for
// sm_100a: "Dense attention is computed only over the top rho K_k blocks".
//
// One CTA = one work item (bh, query cluster a, pair of 128-row query tiles of a).  Q/K/V are the
// cluster-sorted copies [BH, N, d] (bf16).  The kept key clusters of a are packed densely into
// 128-key tiles made of 16 units of 8 consecutive sorted rows; each run of row-contiguous units
// (the units of one cluster inside a tile) is fetched with the fewest TMA boxes (heights 8..128
// rows, one 1 KB SWIZZLE_128B atom per 8 rows), so padding is < 8 rows per kept cluster.  Rows of
// a cluster's last unit past its end are masked to -inf in the softmax.
//
// Warp roles (352 threads):  warps 0-3 softmax/epilogue of Q tile 0 (TMEM lanes 0-127),
// warps 4-7 the same for Q tile 1, warp 8 TMA producer (Q, K), warp 9 TMEM allocator + MMA
// issuer, warp 10 TMA producer (V).
// TMEM (512 cols): S0 [0,128) S1 [128,256) O0 [256,384) O1 [384,512).  P (bf16x2) of keys 0-95
// overwrites the first 48 columns of its S buffer and feeds the PV MMA from TMEM (A operand); P of
// keys 96-127 goes to a per-set SMEM buffer (K-major SWIZZLE_64B) and feeds the last two PV K-steps
// as SS MMAs; V from SMEM (MN-major).  K and V have separate 2-slot rings: K(j) is released as
// soon as both QK(j) MMAs complete and V(j) after both PV(j), so each is prefetched ~2 tiles ahead.
// MMA issue order per KV tile j:  PV0(j)[0-95], QK0(j+1), PV0(j)[96-127], PV1(j)[0-95], QK1(j+1),
// PV1(j)[96-127] — the softmax of one Q tile overlaps the MMAs of the other (FA4-style
// ping-pong), and QK(j+1) no longer waits for the exponentials of the last key quarter of tile j.
// Online softmax in the exp2 domain with lazy rescaling (only when the running max grows by > 8,
// i.e. a factor 256).
// The inverse permutation is fused into the epilogue: row r of the tile is stored as 16-byte
// vectors to O[b, h, perm_q[p], :] in original token order.
#include "kernels.cuh"

namespace cs {
namespace attn {

#ifdef CS_ATTN_DEBUG
// event trace of one CTA (blockIdx 0,0): t[event][tile] = clock64 (debug variant only)
__device__ long long g_trace[20][4096];
// per-CTA timeline (debug variant): [cta][0] entry globaltimer, [1] after setup, [2] first S seen,
// [3] exit, [4] smid, [5] nt, [6] clock64 at entry, [7] clock64 at exit
__device__ long long g_cta[65536][8];
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ int smid() {
  int s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  return s;
}
#define CS_CTA(e, v) \
  if (threadIdx.x == 0 && blockIdx.y * gridDim.x + blockIdx.x < 65536) g_cta[blockIdx.y * gridDim.x + blockIdx.x][e] = (v)
#define CS_CTA_W(e, v) \
  if ((threadIdx.x & 31) == 0 && blockIdx.y * gridDim.x + blockIdx.x < 65536) g_cta[blockIdx.y * gridDim.x + blockIdx.x][e] = (v)
#ifdef CS_ATTN_TRACE  // per-event trace of CTA (0, 0): a branch + clock64 in the hot loop of every CTA
#define CS_TRACE(e, j) \
  if (blockIdx.x == 0 && blockIdx.y == 0 && (threadIdx.x & 31) == 0 && (j) < 4096) g_trace[e][j] = clock64()
#else
#define CS_TRACE(e, j)
#endif
#else
#define CS_TRACE(e, j)
#define CS_CTA(e, v)
#define CS_CTA_W(e, v)
#endif

constexpr int BM = 128, BN = 128, NST = 2;
constexpr int NTHREADS = 352;
constexpr int WARP_PRODUCER = 8, WARP_MMA = 9, WARP_VLOAD = 10;
constexpr float kRescaleThresh = 8.0f;
#ifndef CS_POLY_EVERY
#define CS_POLY_EVERY 4
#endif
constexpr int kPolyEvery = CS_POLY_EVERY;  // one exp2 pair in kPolyEvery on the FMA pipe (0: none)

template <int D>
struct Smem {
  static constexpr int HALVES = D / 64;
  static constexpr int QT = BM * D * 2;   // bytes per Q tile
  static constexpr int KT = BN * D * 2;   // bytes per K (or V) tile
  static constexpr int HALF_Q = BM * 128;  // bytes per 64-col half of a Q tile
  static constexpr int HALF_K = BN * 128;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + 2 * QT;
  static constexpr int OFF_V = OFF_K + NST * KT;
  // P of the last 32 keys of a tile, per accumulator set, K-major SWIZZLE_64B (128 rows x 64 B):
  // the A operand of the two SS MMAs that finish PV(j) after QK(j+1) has been issued
  static constexpr int PLT = BM * 64;
  static constexpr int OFF_PL = OFF_V + NST * KT;
  static constexpr int OFF_BAR = OFF_PL + 2 * PLT;
  // q_full, k_full[2], k_empty[2], v_full[2], v_empty[2], s_full[2], p_full[2 sets][3 parts], o_full,
  // pvd[2]
  static constexpr int OFF_MISC = OFF_BAR + 24 * 8;  // tmem slot, R, n
  static constexpr int OFF_KSTART = OFF_MISC + 16;    // [n] first sorted row of kept cluster i
  static constexpr int OFF_RCUM = OFF_KSTART + kMaxClusters * 4;  // [n + 1] row prefix sums
  static constexpr int OFF_XCH = OFF_RCUM + ((kMaxClusters + 1) * 4 + 15) / 16 * 16;
  static constexpr int BYTES = OFF_XCH + 4 * BM * 4;  // split-KV merge: m[2][BM], l[2][BM]
  static constexpr int ALLOC = BYTES + 1024;  // room to align the base to 1024
};

template <int D>
__global__ void __launch_bounds__(NTHREADS, 1)
    k_bsa_fwd(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ KVMaps kv, int H, int N,
              int kq, int kk, const int32_t* __restrict__ perm_q, const int32_t* __restrict__ offs_q,
              const int32_t* __restrict__ offs_k, const int32_t* __restrict__ n_keep,
              const int32_t* __restrict__ n_rows, const int32_t* __restrict__ kept,
              const int32_t* __restrict__ item_start,
              float scale_log2, __nv_bfloat16* __restrict__ out, long long osb, long long osh,
              long long osn, const uint64_t* __restrict__ peer_ptrs, int peer_npr, int peer_head_base) {
  using L = Smem<D>;
  extern __shared__ uint8_t smem_raw[];
  // align to 1024 B while keeping the pointer in the shared window (LDS/STS, not generic LD/ST)
  uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L::OFF_BAR);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;
  uint64_t* k_empty = bars + 3;
  uint64_t* v_full = bars + 5;
  uint64_t* v_empty = bars + 7;
  uint64_t* s_full = bars + 9;
  uint64_t* p_full = bars + 11;  // [tq * 3 + part]: P of keys 0-63 / 64-95 (TMEM), 96-127 (SMEM)
  uint64_t* o_full = bars + 17;
  uint64_t* pvd = bars + 18;     // [tq]: PV(j) of set tq complete (its SMEM part included)
  int* misc = reinterpret_cast<int*>(sm + L::OFF_MISC);
  int* kstart = reinterpret_cast<int*>(sm + L::OFF_KSTART);
  int* rcum = reinterpret_cast<int*>(sm + L::OFF_RCUM);
  float* xch = reinterpret_cast<float*>(sm + L::OFF_XCH);

  CS_CTA(0, gtimer());
  CS_CTA(6, clock64());
  const int bh = blockIdx.y;
  const int item = blockIdx.x;
  const int32_t* ist = item_start + (size_t)bh * (kq + 1);
  if (item >= ist[kq]) return;  // uniform across the CTA
  // query cluster a: largest a with ist[a] <= item
  int lo = 0, hi = kq - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (ist[mid] <= item) lo = mid; else hi = mid - 1;
  }
  const int a = lo;
  const int pair = item - ist[a];
  const int qbeg = offs_q[(size_t)bh * (kq + 1) + a];
  const int qlen = offs_q[(size_t)bh * (kq + 1) + a + 1] - qbeg;
  const int t0 = 2 * pair;
  const bool has1 = (t0 + 1) * BM < qlen;
  // single-tile item: split the KV sequence between the two accumulator sets (even / odd KV
  // tiles) so the softmax of one still overlaps the MMAs of the other; merged in the epilogue
  const bool split = !has1;
  const int warp = warp_id(), lane = lane_id();

  // ---- setup: barriers + Q load (warp 8, lane 0: the Q tiles do not depend on the unit table, so
  // their TMA is in flight while the table is built), TMEM (warp 9), unit table (warp 8)
  if (warp == WARP_PRODUCER) {
    if (lane == 0) {
      mbar_init(q_full, 1);
      for (int s = 0; s < NST; ++s) {
        mbar_init(k_full + s, 1); mbar_init(k_empty + s, 1);
        mbar_init(v_full + s, 1); mbar_init(v_empty + s, 1);
      }
      for (int t = 0; t < 2; ++t) mbar_init(s_full + t, 1);
      for (int t = 0; t < 6; ++t) mbar_init(p_full + t, 128);
      mbar_init(o_full, 1);
      for (int t = 0; t < 2; ++t) mbar_init(pvd + t, 1);
      fence_barrier_init();
      tma_prefetch_desc(&tm_q);
      const int ntq = has1 ? 2 : 1;
      mbar_arrive_expect_tx(q_full, ntq * L::QT);
      for (int tq = 0; tq < ntq; ++tq)
        for (int hf = 0; hf < L::HALVES; ++hf)
          tma_load_2d(sm + L::OFF_Q + tq * L::QT + hf * L::HALF_Q, &tm_q, hf * 64,
                      bh * N + qbeg + (t0 + tq) * BM, q_full);
    }
    if (lane < kKVBoxes) { tma_prefetch_desc(&kv.k[lane]); tma_prefetch_desc(&kv.v[lane]); }
  }
  if (warp == WARP_MMA) {
    tmem_alloc(reinterpret_cast<uint32_t*>(misc), 512);

  }
  if (warp == WARP_PRODUCER) {
    const int n = n_rows ? n_rows[(size_t)bh * kq + a] : n_keep[bh];  // per-row counts (R11b)
    const int32_t* kl = kept + ((size_t)bh * kq + a) * kk;
    const int32_t* ok = offs_k + (size_t)bh * (kk + 1);
    int carry = 0;
    // 4 chunks of 32 kept clusters per round: all kept-list loads, then all offset loads, in
    // flight together (two dependent global-load rounds per 128 clusters)
    for (int i0 = 0; i0 < n; i0 += 128) {
      int c4[4], st4[4], en4[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + 32 * u + lane;
        c4[u] = i < n ? kl[i] : 0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + 32 * u + lane;
        st4[u] = i < n ? ok[c4[u]] : 0;
        en4[u] = i < n ? ok[c4[u] + 1] : 0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + 32 * u + lane;
        const int len = i < n ? en4[u] - st4[u] : 0;
        if (i < n) kstart[i] = st4[u];
        int x = len;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) { int y = __shfl_up_sync(0xffffffffu, x, o); if (lane >= o) x += y; }
        if (i < n) rcum[i] = carry + x - len;
        carry += __shfl_sync(0xffffffffu, x, 31);
      }
    }
    if (lane == 0) { rcum[n] = carry; misc[1] = carry; misc[2] = n; }

  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = static_cast<uint32_t>(misc[0]);
  const int R = misc[1];  // kept key rows, packed back to back into 128-key tiles
  const int nkeep = misc[2];
  const int nt = (R + BN - 1) / BN;
  CS_CTA(1, gtimer());
  CS_CTA(4, smid());
  CS_CTA(5, nt | (split ? (1 << 20) : 0));

  if (warp == WARP_PRODUCER || warp == WARP_VLOAD) {
    // ================= TMA producers: warp 8 -> Q and K(j), warp 10 -> V(j) =================
    const bool is_v = warp == WARP_VLOAD;
    // Tile jj holds the kept rows [BN jj, BN jj + BN) of the concatenation of the kept clusters (in
    // ascending cluster order).  Lane l takes the l-th cluster overlapping the tile (32 at a time)
    // and issues the power-of-two row boxes (8..128 and 1..7 rows x 64 columns, SWIZZLE_128B: a box written
    // at any 128-byte row offset lands in the tile's swizzled layout, scripts/micro/
    // tma_rowbox_test.cu) that cover its segment; the last tile's rows past R are filled from the
    // head's first rows (finite values; masked to -inf in the softmax).
    int cur = 0;  // first kept cluster overlapping the current tile (warp-uniform)
    auto issue_tile = [&](uint64_t* bar, uint8_t* base, int jj) {
      const int t_beg = jj * BN, t_end = t_beg + BN;
      if (lane == 0) mbar_arrive_expect_tx(bar, L::KT);
      __syncwarp();
      // boxes of 128 .. 8 rows (maps 4 .. 0) for the multiple of 8, one box of 1..7 rows (map 4 + r)
      // for the remainder
      auto boxes = [&](int trow, int grow, int len) {
        int off = 0;
#pragma unroll 1
        for (int bi = 4; bi >= 0; --bi) {
          if (len & (8 << bi)) {
#pragma unroll
            for (int hf = 0; hf < L::HALVES; ++hf)
              tma_load_2d(base + hf * L::HALF_K + (trow + off) * 128, is_v ? &kv.v[bi] : &kv.k[bi], hf * 64, grow + off, bar);
            off += 8 << bi;
          }
        }
        if (len & 7) {
          const int bi = 4 + (len & 7);
#pragma unroll
          for (int hf = 0; hf < L::HALVES; ++hf)
            tma_load_2d(base + hf * L::HALF_K + (trow + off) * 128, is_v ? &kv.v[bi] : &kv.k[bi], hf * 64, grow + off, bar);
        }
      };
      while (cur < nkeep && rcum[cur + 1] <= t_beg) ++cur;
      for (int i0 = cur; i0 < nkeep && rcum[i0] < t_end; i0 += 32) {
        const int i = i0 + lane;
        if (i < nkeep && rcum[i] < t_end) {
          const int s0 = max(rcum[i], t_beg), s1 = min(rcum[i + 1], t_end);
          if (s1 > s0) boxes(s0 - t_beg, bh * N + kstart[i] + (s0 - rcum[i]), s1 - s0);
        }
      }
      if (lane == 0 && t_end > R) boxes(R - t_beg, bh * N, t_end - R);
      __syncwarp();
    };
    uint64_t* full = is_v ? v_full : k_full;
    uint64_t* empty = is_v ? v_empty : k_empty;
    uint8_t* ring = sm + (is_v ? L::OFF_V : L::OFF_K);
    for (int jj = 0; jj < nt; ++jj) {
      const int slot = jj % NST;
      mbar_wait(empty + slot, ((jj / NST) & 1) ^ 1);
      if (lane == 0) CS_TRACE(is_v ? 10 : 9, jj);
      issue_tile(full + slot, ring + slot * L::KT, jj);
      if (lane == 0) CS_TRACE(is_v ? 1 : 0, jj);
    }
  } else if (warp == WARP_MMA) {
    // ================= MMA issuer (whole warp, one elected lane issues) =================
    // Descriptors are built once; inside the loop a K-step or a ring slot is a constant offset
    // added to the 14-bit start-address field (addresses stay < 256 KB, so no carry out).
    constexpr uint32_t idesc_qk = idesc_bf16(BM, BN, 0, 0);
    constexpr uint32_t idesc_pv = idesc_bf16(BM, D, 0, 1);
    const uint64_t dq0 = smem_desc_sw128(smem_u32(sm + L::OFF_Q), 16, 1024);
    const uint64_t dk0 = smem_desc_sw128(smem_u32(sm + L::OFF_K), 16, 1024);
    const uint64_t dv0 = smem_desc_sw128(smem_u32(sm + L::OFF_V), L::HALF_K, 1024);
    auto issue_qk = [&](int tq, int slot, int qs) {  // S[tq] = Q slot qs x K slot `slot`
      if (elect_one()) {
        const uint32_t d_tmem = tmem + tq * 128;
        const uint64_t qd = dq0 + (uint64_t)((qs * L::QT) >> 4);
        const uint64_t kd = dk0 + (uint64_t)((slot * L::KT) >> 4);
#pragma unroll
        for (int kk2 = 0; kk2 < D / 16; ++kk2) {
          const uint32_t off = ((kk2 >> 2) * L::HALF_Q + (kk2 & 3) * 32) >> 4;
          const uint32_t offk = ((kk2 >> 2) * L::HALF_K + (kk2 & 3) * 32) >> 4;
          mma_ss(d_tmem, qd + off, kd + offk, idesc_qk, kk2 > 0);
        }
      }
      __syncwarp();
    };
    // PV(j) in three parts: K-steps [k0, k1) with P from TMEM (keys 0-95, 6 K-steps), then keys
    // 96-127 with P from SMEM (SS form, 2 K-steps) once QK(j+1) has been issued: QK(j+1) overwrites
    // the TMEM columns of P, so it may only follow the TMEM parts of PV(j), and the last quarter of
    // the exponentials no longer sits between S(j) and S(j+1).
    auto issue_pv_tmem = [&](int tq, int slot, int k0, int k1, bool acc) {
      if (elect_one()) {
        const uint32_t d_tmem = tmem + 256 + tq * 128;
        const uint32_t p_tmem = tmem + tq * 128;
        const uint64_t vd = dv0 + (uint64_t)((slot * L::KT) >> 4);
        for (int kk2 = k0; kk2 < k1; ++kk2)
          mma_ts(d_tmem, p_tmem + kk2 * 8, vd + (uint64_t)((kk2 * 2048) >> 4), idesc_pv, (acc || kk2 > 0) ? 1u : 0u);
      }
      __syncwarp();
    };
    auto issue_pv_smem = [&](int tq, int slot) {
      if (elect_one()) {
        const uint32_t d_tmem = tmem + 256 + tq * 128;
        const uint64_t pd = smem_desc_sw64(smem_u32(sm + L::OFF_PL + tq * L::PLT), 512);
        const uint64_t vd = dv0 + (uint64_t)((slot * L::KT) >> 4);
#pragma unroll
        for (int kk2 = 6; kk2 < 8; ++kk2)
          mma_ss(d_tmem, pd + (uint64_t)(((kk2 - 6) * 32) >> 4), vd + (uint64_t)((kk2 * 2048) >> 4), idesc_pv, 1u);
      }
      __syncwarp();
    };
    auto commit = [&](uint64_t* bar) {
      if (elect_one()) mma_commit(bar);
      __syncwarp();
    };
    auto pv_early = [&](int tq, int slot, int j) {
      mbar_wait(p_full + tq * 3 + 0, j & 1);
      tc_fence_after();
      issue_pv_tmem(tq, slot, 0, 4, j > 0);
      mbar_wait(p_full + tq * 3 + 1, j & 1);
      tc_fence_after();
      issue_pv_tmem(tq, slot, 4, 6, true);
    };
    auto pv_late = [&](int tq, int slot, int j) {
      mbar_wait(p_full + tq * 3 + 2, j & 1);
      tc_fence_after();
      issue_pv_smem(tq, slot);
      commit(pvd + tq);
    };
    
    mbar_wait(q_full, 0);
    if (nt == 0) {
      // no allowed key (a caller-supplied kept row of empty clusters): nothing to multiply; the
      // softmax warps write zero rows
    } else if (!split) {
      // two Q tiles share every K/V tile.  Per KV tile j: PV0(j), QK0(j+1), PV1(j), QK1(j+1).
      mbar_wait(k_full, 0);
      tc_fence_after();
      issue_qk(0, 0, 0);
      commit(s_full + 0);
      if (has1) { issue_qk(1, 0, 1); commit(s_full + 1); }
      commit(k_empty + 0);
      for (int j = 0; j < nt; ++j) {
        const int slot = j % NST, slot1 = (j + 1) % NST;
        const bool more = j + 1 < nt;
        mbar_wait(v_full + slot, (j / NST) & 1);
        CS_TRACE(3, j);
        pv_early(0, slot, j);
        CS_TRACE(4, j);
        if (more) {
          mbar_wait(k_full + slot1, ((j + 1) / NST) & 1);
          CS_TRACE(2, j + 1);
          tc_fence_after();
          issue_qk(0, slot1, 0);
          commit(s_full + 0);
        }
        pv_late(0, slot, j);
        if (has1) {
          pv_early(1, slot, j);
          CS_TRACE(11, j);
          if (more) { issue_qk(1, slot1, 1); commit(s_full + 1); }
          pv_late(1, slot, j);
        }
        commit(v_empty + slot);
        if (more) commit(k_empty + slot1);
      }
    } else {
      // split-KV: one Q tile (slot 0); accumulator set tq takes the KV tiles 2j + tq, which the
      // producers place in ring slot tq (use j of the slot -> parity j & 1).  Same ping-pong:
      // PV0(2j), QK0(2j+2), PV1(2j+1), QK1(2j+3).
      mbar_wait(k_full + 0, 0);
      tc_fence_after();
      issue_qk(0, 0, 0);
      commit(s_full + 0);
      commit(k_empty + 0);
      if (nt > 1) {
        mbar_wait(k_full + 1, 0);
        tc_fence_after();
        issue_qk(1, 1, 0);
        commit(s_full + 1);
        commit(k_empty + 1);
      }
      for (int j = 0; 2 * j < nt; ++j) {
        const bool has_b = 2 * j + 1 < nt, more_a = 2 * j + 2 < nt, more_b = 2 * j + 3 < nt;
        mbar_wait(v_full + 0, j & 1);
        pv_early(0, 0, j);
        if (more_a) {
          mbar_wait(k_full + 0, (j + 1) & 1);
          tc_fence_after();
          issue_qk(0, 0, 0);
          commit(s_full + 0);
          commit(k_empty + 0);
        }
        pv_late(0, 0, j);
        commit(v_empty + 0);
        if (has_b) {
          mbar_wait(v_full + 1, j & 1);
          pv_early(1, 1, j);
          if (more_b) {
            mbar_wait(k_full + 1, (j + 1) & 1);
            tc_fence_after();
            issue_qk(1, 1, 0);
            commit(s_full + 1);
            commit(k_empty + 1);
          }
          pv_late(1, 1, j);
          commit(v_empty + 1);
        }
      }
    }
    commit(o_full);
  } else {
    // ================= softmax / epilogue (warps 0-7) =================
    const int tq = warp >> 2;
    // KV tiles of this accumulator set: all of them, or every other one (from tq) when split
    const int my_nt = split ? (nt + 1 - tq) / 2 : nt;
    // output row of this thread: its token, and the destination row in original token order (or
    // in the owning peer's block when the Ulysses return is fused)
    auto out_row = [&](int prow, bool& row_ok) -> __nv_bfloat16* {
      row_ok = prow < qlen;
      const int tok = row_ok ? perm_q[(size_t)bh * N + qbeg + prow] : 0;
      const int b = bh / H, h = bh % H;
      if (peer_ptrs) {
        // fused Ulysses return all-to-all: token tok lives on rank tok / npr, whose [N/P, H_total,
        // d] token block is mapped into this process (NVLink P2P / CUDA IPC); head h of this call
        // is global head peer_head_base + h.  The 16-byte row stores go straight to the peer.
        const int pr = tok / peer_npr;
        return reinterpret_cast<__nv_bfloat16*>(peer_ptrs[pr]) + (long long)(tok - pr * peer_npr) * osn +
               (long long)(peer_head_base + h) * osh;
      }
      return out + (long long)b * osb + (long long)h * osh + (long long)tok * osn;
    };
    if (nt == 0 && (tq == 0 || has1)) {
      // empty allowed key set: defined result o_i = 0
      bool row_ok;
      uint4* d4 = reinterpret_cast<uint4*>(out_row(t0 * BM + tq * BM + (warp & 3) * 32 + lane, row_ok));
      if (row_ok)
#pragma unroll
        for (int i = 0; i < D / 8; ++i) d4[i] = make_uint4(0u, 0u, 0u, 0u);
    }
    if (my_nt > 0) {
      const int quad = warp & 3;
      const int r = quad * 32 + lane;  // row of the Q tile == TMEM lane
      const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
      const uint32_t s_tm = tmem + lane_off + tq * 128;
      const uint32_t o_tm = tmem + lane_off + 256 + tq * 128;
      float m = -INFINITY, l = 0.f;
      // invalid columns: only the last tile's, past the R kept rows (the tiles are row-exact)
      uint32_t mw0 = 0, mw1 = 0, mw2 = 0, mw3 = 0;
      auto tile_mask = [&](int j) {
        const int v = R - j * BN;  // valid columns of tile j
        auto word = [&](int w) -> uint32_t {
          const int c = v - 32 * w;
          return c >= 32 ? 0u : (c <= 0 ? 0xffffffffu : (0xffffffffu << c));
        };
        mw0 = word(0); mw1 = word(1); mw2 = word(2); mw3 = word(3);
      };
      tile_mask(split ? tq : 0);
      for (int j = 0; j < my_nt; ++j) {
        mbar_wait(s_full + tq, j & 1);
        CS_TRACE(5 + 2 * tq, j);
        if (j == 0 && warp == 0) CS_CTA(2, gtimer());
        tc_fence_after();
#define CS_APPLY_MASK(W, MWV)                                                        \
  if (MWV) {                                                                         \
    _Pragma("unroll") for (int r2 = 0; r2 < 32; ++r2) if ((MWV >> r2) & 1u) su[W * 32 + r2] = 0xff800000u; \
  }
        uint32_t su[BN];
#pragma unroll
        for (int c = 0; c < BN / 32; ++c) tmem_ld32(s_tm + c * 32, su + c * 32);
        tmem_wait_ld();
        CS_APPLY_MASK(0, mw0)
        CS_APPLY_MASK(1, mw1)
        CS_APPLY_MASK(2, mw2)
        CS_APPLY_MASK(3, mw3)
        CS_TRACE(16 + tq, j);
        // row max of the raw scores: 8 independent 3-input max chains
        float mx8[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) mx8[i] = fmaxf(__uint_as_float(su[i]), __uint_as_float(su[8 + i]));
#pragma unroll
        for (int c = 16; c < BN; c += 16)
#pragma unroll
          for (int i = 0; i < 8; ++i) mx8[i] = fmax3(mx8[i], __uint_as_float(su[c + i]), __uint_as_float(su[c + 8 + i]));
        const float mx = fmax3(fmax3(mx8[0], mx8[1], mx8[2]), fmax3(mx8[3], mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])) *
                         scale_log2;
        CS_TRACE(12 + tq, j);
        float alpha = 1.f;
        if (j == 0) {
          m = mx;
        } else if (mx > m + kRescaleThresh) {
          alpha = ex2(m - mx);
          l *= alpha;
          m = mx;
        }
        const bool warp_rescale = __any_sync(0xffffffffu, alpha != 1.f);
        // p = 2^(s*scale_log2 - m): paired FFMA2, MUFU ex2, 4 independent FADD2 row-sum chains.
        // P is stored and signalled in three parts (keys 0-63 and 64-95 to TMEM, 96-127 to SMEM):
        // PV on the first part overlaps the exponentials of the rest, and QK(j+1) is issued as
        // soon as the TMEM parts have been consumed.
        const float2 sl2 = make_float2(scale_log2, scale_log2), nm2 = make_float2(-m, -m);
        float2 acc4[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
        // exponentials of keys [c0, c1), packed in place over su[c0 / 2 ..): every kPolyEvery-th pair
        // on the FMA pipe (polynomial), the rest on MUFU
        auto exp_range = [&](int c0, int c1) {
#pragma unroll
          for (int c = c0; c < c1; c += 2) {
            const float2 x = ffma2(make_float2(__uint_as_float(su[c]), __uint_as_float(su[c + 1])), sl2, nm2);
            const float2 p = (kPolyEvery > 0 && ((c >> 1) % kPolyEvery) == kPolyEvery - 1)
                                 ? ex2_poly2(x) : make_float2(ex2(x.x), ex2(x.y));
            acc4[(c >> 1) & 3] = fadd2(acc4[(c >> 1) & 3], p);
            su[c >> 1] = pack_bf16x2(p.x, p.y);
          }
        };
        // part A: keys 0-63 -> TMEM columns 0-31
        exp_range(0, 64);
        tmem_st32(s_tm, su);
        // lazy O rescale before PV(j) starts (it waits for p_full(j, part A)).  tcgen05.ld/st are
        // warp-collective, so the warp rescales if any of its rows needs it.  O is stable once the
        // SMEM part of PV(j-1) completed (pvd): the TMEM parts precede s_full(j) in commit order.
        if (warp_rescale) {
          if (j > 0) mbar_wait(pvd + tq, (j - 1) & 1);
          tc_fence_after();
#pragma unroll 1
          for (int c = 0; c < D / 16; ++c) {
            uint32_t ov[16];
            tmem_ld16(o_tm + c * 16, ov);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * alpha);
            tmem_st16(o_tm + c * 16, ov);
          }
        }
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(p_full + tq * 3 + 0);
        CS_TRACE(14 + tq, j);
        // part B: keys 64-95 -> TMEM columns 32-47 (QK(j+1) follows its PV)
        exp_range(64, 96);
        tmem_st16(s_tm + 32, su + 32);
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(p_full + tq * 3 + 1);
        // part C: keys 96-127 -> this set's SMEM P buffer (K-major SWIZZLE_64B: 16-byte chunk q of
        // row r at chunk position q ^ ((r >> 1) & 3) of its 64-byte row, 8-row atoms of 512 B),
        // once the SMEM part of PV(j-1) has read the previous contents
        exp_range(96, 128);
        if (j > 0) mbar_wait(pvd + tq, (j - 1) & 1);
        {
          uint8_t* prow = sm + Smem<D>::OFF_PL + tq * Smem<D>::PLT + (r >> 3) * 512 + (r & 7) * 64;
#pragma unroll
          for (int q = 0; q < 4; ++q)
            *reinterpret_cast<uint4*>(prow + ((q ^ ((r >> 1) & 3)) * 16)) =
                make_uint4(su[48 + 4 * q], su[49 + 4 * q], su[50 + 4 * q], su[51 + 4 * q]);
        }
        fence_proxy_async_smem();
        mbar_arrive(p_full + tq * 3 + 2);
        const float2 s01 = fadd2(acc4[0], acc4[1]), s23 = fadd2(acc4[2], acc4[3]);
        const float2 s4 = fadd2(s01, s23);
        l += s4.x + s4.y;
#undef CS_APPLY_MASK
        CS_TRACE(6 + 2 * tq, j);
        if (j + 1 < my_nt) tile_mask(split ? 2 * (j + 1) + tq : j + 1);
      }
      // ---- epilogue: O / l -> bf16, scattered to original token order
      mbar_wait(o_full, 0);
      tc_fence_after();
      bool row_ok;
      __nv_bfloat16* dst = out_row((t0 + (split ? 0 : tq)) * BM + r, row_ok);
      if (split && nt > 1) {
        // merge the two partial states of the row (each relative to its own running max):
        // O = (O0 2^(m0-M) + O1 2^(m1-M)) / (l0 2^(m0-M) + l1 2^(m1-M)); set tq writes the
        // output columns [tq D/2, (tq+1) D/2)
        xch[tq * BM + r] = m;
        xch[(2 + tq) * BM + r] = l;
        named_bar_sync(1, 256);
        const float m0 = xch[r], m1 = xch[BM + r];
        const float M = fmaxf(m0, m1);
        const float a0 = ex2(m0 - M), a1 = ex2(m1 - M);
        const float inv = 1.f / (xch[2 * BM + r] * a0 + xch[3 * BM + r] * a1);
        const float f0 = a0 * inv, f1 = a1 * inv;
        const uint32_t o0 = tmem + lane_off + 256, o1 = tmem + lane_off + 384;
#pragma unroll 1
        for (int c0 = 0; c0 < D / 64; ++c0) {
          const int c = tq * (D / 64) + c0;
          uint32_t u0[32], u1[32];
          tmem_ld32(o0 + c * 32, u0);
          tmem_ld32(o1 + c * 32, u1);
          tmem_wait_ld();
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i)
            pk[i] = pack_bf16x2(__uint_as_float(u0[2 * i]) * f0 + __uint_as_float(u1[2 * i]) * f1,
                                __uint_as_float(u0[2 * i + 1]) * f0 + __uint_as_float(u1[2 * i + 1]) * f1);
          if (row_ok) {
            uint4* d4 = reinterpret_cast<uint4*>(dst + c * 32);
#pragma unroll
            for (int i = 0; i < 4; ++i) d4[i] = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
          }
        }
      } else {
        const float inv_l = 1.f / l;
#pragma unroll
        for (int c = 0; c < D / 32; ++c) {
          uint32_t ov[32];
          tmem_ld32(o_tm + c * 32, ov);
          tmem_wait_ld();
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i)
            pk[i] = pack_bf16x2(__uint_as_float(ov[2 * i]) * inv_l, __uint_as_float(ov[2 * i + 1]) * inv_l);
          if (row_ok) {
            uint4* d4 = reinterpret_cast<uint4*>(dst + c * 32);
#pragma unroll
            for (int i = 0; i < 4; ++i) d4[i] = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
          }
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
  CS_CTA(3, gtimer());
  CS_CTA(7, clock64());
}

}  // namespace attn

#ifdef CS_ATTN_DEBUG
extern "C" int cs_debug_attn_cta(void* host, size_t bytes) {
  return (int)cudaMemcpyFromSymbol(host, attn::g_cta, bytes < sizeof(attn::g_cta) ? bytes : sizeof(attn::g_cta));
}
extern "C" int cs_debug_attn_trace(void* host, size_t bytes) {
  return (int)cudaMemcpyFromSymbol(host, attn::g_trace, bytes < sizeof(attn::g_trace) ? bytes : sizeof(attn::g_trace));
}
#endif

cudaError_t launch_bsa_fwd(const CUtensorMap* tm_q, const KVMaps* kv,
                           int BH, int H, int N, int d, int kq, int kk, const int32_t* perm_q,
                           const int32_t* offs_q, const int32_t* offs_k, const int32_t* n_keep,
                           const int32_t* n_rows, const int32_t* kept, const int32_t* item_start, int items_ub,
                           float scale, __nv_bfloat16* o, long long osb, long long osh,
                           long long osn, const uint64_t* peer_ptrs, int peer_npr, int peer_head_base,
                           cudaStream_t st) {
  const float scale_log2 = scale * 1.4426950408889634f;
  dim3 grid(items_ub, BH);
  if (d == 128) {
    auto kfn = attn::k_bsa_fwd<128>;
    const int smem = attn::Smem<128>::ALLOC;
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    kfn<<<grid, attn::NTHREADS, smem, st>>>(*tm_q, *kv, H, N, kq, kk, perm_q, offs_q, offs_k,
                                           n_keep, n_rows, kept, item_start, scale_log2, o, osb, osh, osn,
                                           peer_ptrs, peer_npr, peer_head_base);
  } else {
    auto kfn = attn::k_bsa_fwd<64>;
    const int smem = attn::Smem<64>::ALLOC;
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    kfn<<<grid, attn::NTHREADS, smem, st>>>(*tm_q, *kv, H, N, kq, kk, perm_q, offs_q, offs_k,
                                           n_keep, n_rows, kept, item_start, scale_log2, o, osb, osh, osn,
                                           peer_ptrs, peer_npr, peer_head_base);
  }
  return cudaGetLastError();
}

}  // namespace cs
