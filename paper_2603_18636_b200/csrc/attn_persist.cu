// attn_persist.cu — the block-sparse attention of attn.cu as a PERSISTENT kernel:
// one CTA per SM walks the work items (bh, query cluster a, pair of 128-row query tiles)
// c, c + G, c + 2G, ... of the head-major item space, so one item's prologue overlaps the previous
// item's tail instead of paying a CTA launch, barrier / TMEM setup and cold pipeline per item.
//
// Same warp roles, tiles, TMEM map, softmax and epilogue as attn.cu (see its header).  What the
// persistence adds:
//  * the unit table (kept clusters -> sorted rows) is double-buffered: the producer builds item
//    i+1's table while item i still computes (tab_full / tab_free barriers per buffer);
//  * the Q tiles of item i+1 are loaded as soon as the last QK of item i completes (q_empty);
//  * the K / V rings and the S / P barriers keep running use counters across items;
//  * the first PV of item i+1 (which overwrites O) waits until every softmax thread has read item
//    i's O in its epilogue (o_free), so the next item's first QK and softmax overlap that epilogue.
#include "kernels.cuh"

namespace cs {
namespace attn_p {

constexpr int BM = 128, BN = 128, UNIT = 8, UPT = BN / UNIT, NST = 2;
constexpr int NTHREADS = 352;
constexpr int WARP_PRODUCER = 8, WARP_MMA = 9, WARP_VLOAD = 10;
constexpr float kRescaleThresh = 8.0f;
constexpr int kPolyEvery = 4;
constexpr int TAB_CONSUMERS = 10;  // lane 0 of: 8 softmax warps, the MMA warp, the V producer

template <int D>
struct Smem {
  static constexpr int HALVES = D / 64;
  static constexpr int QT = BM * D * 2, KT = BN * D * 2;
  static constexpr int HALF_Q = BM * 128, HALF_K = BN * 128;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + 2 * QT;
  static constexpr int OFF_V = OFF_K + NST * KT;
  static constexpr int OFF_BAR = OFF_V + NST * KT;
  // q_full, q_empty, k_full[2], k_empty[2], v_full[2], v_empty[2], s_full[2], p_full[4], o_full,
  // o_free, tab_full[2], tab_free[2]
  static constexpr int NBAR = 22;
  static constexpr int OFF_MISC = OFF_BAR + NBAR * 8 + 16;          // tmem slot
  // unit tables, double-buffered: kstart[kMax], klen[kMax], ucum[kMax+1], meta {U, nkeep}
  static constexpr int TAB_INTS = 3 * kMaxClusters + 1 + 3;
  static constexpr int OFF_TAB = (OFF_MISC + 16 + 15) / 16 * 16;
  static constexpr int OFF_XCH = OFF_TAB + ((2 * TAB_INTS * 4 + 15) / 16) * 16;
  static constexpr int BYTES = OFF_XCH + 4 * BM * 4;
  static constexpr int ALLOC = BYTES + 1024;
};

struct Item {
  int bh, a, pair, qbeg, qlen, t0;
  bool has1, split;
};

// next valid item of this CTA's slot sequence (identical in every role)
__device__ __forceinline__ bool next_item(int& slot, int total_slots, int items_ub, int kq,
                                          const int32_t* __restrict__ item_start,
                                          const int32_t* __restrict__ offs_q, Item& it) {
  while (slot < total_slots) {
    const int bh = slot / items_ub, item = slot % items_ub;
    slot += gridDim.x;
    const int32_t* ist = item_start + (size_t)bh * (kq + 1);
    if (item >= ist[kq]) continue;
    int lo = 0, hi = kq - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (ist[mid] <= item) lo = mid; else hi = mid - 1;
    }
    it.bh = bh;
    it.a = lo;
    it.pair = item - ist[lo];
    it.qbeg = offs_q[(size_t)bh * (kq + 1) + lo];
    it.qlen = offs_q[(size_t)bh * (kq + 1) + lo + 1] - it.qbeg;
    it.t0 = 2 * it.pair;
    it.has1 = (it.t0 + 1) * BM < it.qlen;
    it.split = !it.has1;
    return true;
  }
  return false;
}

template <int D>
__global__ void __launch_bounds__(NTHREADS, 1)
    k_bsa_fwd_persist(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ KVMaps kv, int H,
                      int N, int kq, int kk, const int32_t* __restrict__ perm_q,
                      const int32_t* __restrict__ offs_q, const int32_t* __restrict__ offs_k,
                      const int32_t* __restrict__ n_keep, const int32_t* __restrict__ n_rows,
                      const int32_t* __restrict__ kept, const int32_t* __restrict__ item_start,
                      int items_ub, int total_slots, float scale_log2, __nv_bfloat16* __restrict__ out,
                      long long osb, long long osh, long long osn, const uint64_t* __restrict__ peer_ptrs,
                      int peer_npr, int peer_head_base) {
  using L = Smem<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L::OFF_BAR);
  uint64_t* q_full = bars;
  uint64_t* q_empty = bars + 1;
  uint64_t* k_full = bars + 2;
  uint64_t* k_empty = bars + 4;
  uint64_t* v_full = bars + 6;
  uint64_t* v_empty = bars + 8;
  uint64_t* s_full = bars + 10;
  uint64_t* p_full = bars + 12;  // [tq * 2 + half]
  uint64_t* o_full = bars + 16;
  uint64_t* o_free = bars + 17;
  uint64_t* tab_full = bars + 18;
  uint64_t* tab_free = bars + 20;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + L::OFF_MISC);
  int* tabs = reinterpret_cast<int*>(sm + L::OFF_TAB);
  float* xch = reinterpret_cast<float*>(sm + L::OFF_XCH);
  auto tab_kstart = [&](int b) { return tabs + b * L::TAB_INTS; };
  auto tab_klen = [&](int b) { return tabs + b * L::TAB_INTS + kMaxClusters; };
  auto tab_ucum = [&](int b) { return tabs + b * L::TAB_INTS + 2 * kMaxClusters; };
  auto tab_meta = [&](int b) { return tabs + b * L::TAB_INTS + 3 * kMaxClusters + 1; };

  const int warp = warp_id(), lane = lane_id();
  if (warp == WARP_PRODUCER && lane == 0) {
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int s = 0; s < NST; ++s) {
      mbar_init(k_full + s, 1); mbar_init(k_empty + s, 1);
      mbar_init(v_full + s, 1); mbar_init(v_empty + s, 1);
    }
    for (int t = 0; t < 2; ++t) mbar_init(s_full + t, 1);
    for (int t = 0; t < 4; ++t) mbar_init(p_full + t, 128);
    mbar_init(o_full, 1);
    mbar_init(o_free, 256);
    for (int t = 0; t < 2; ++t) { mbar_init(tab_full + t, 1); mbar_init(tab_free + t, TAB_CONSUMERS); }
    fence_barrier_init();
  }
  if (warp == WARP_PRODUCER) {
    tma_prefetch_desc(&tm_q);
    if (lane < 5) { tma_prefetch_desc(&kv.k[lane]); tma_prefetch_desc(&kv.v[lane]); }
  }
  if (warp == WARP_MMA) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  int slot = blockIdx.x;
  Item it;

  if (warp == WARP_PRODUCER || warp == WARP_VLOAD) {
    // ================= TMA producers: warp 8 -> tables, Q and K(j); warp 10 -> V(j) =========
    const bool is_v = warp == WARP_VLOAD;
    uint64_t* full = is_v ? v_full : k_full;
    uint64_t* empty = is_v ? v_empty : k_empty;
    uint8_t* ring = sm + (is_v ? L::OFF_V : L::OFF_K);
    int use[2] = {0, 0};  // ring slot use counters (across items)
    for (int li = 0; next_item(slot, total_slots, items_ub, kq, item_start, offs_q, it); ++li) {
      const int tb = li & 1;
      int* kstart = tab_kstart(tb);
      int* klen = tab_klen(tb);
      int* ucum = tab_ucum(tb);
      int* meta = tab_meta(tb);
      const int bh = it.bh;
      if (!is_v) {
        // table of this item into buffer tb (free once every consumer is done with item li-2)
        if (li >= 2) mbar_wait(tab_free + tb, ((li >> 1) - 1) & 1);
        const int n = n_rows ? n_rows[(size_t)bh * kq + it.a] : n_keep[bh];
        const int32_t* kl = kept + ((size_t)bh * kq + it.a) * kk;
        const int32_t* ok = offs_k + (size_t)bh * (kk + 1);
        int carry = 0;
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
            const int len = en4[u] - st4[u];
            const int nu = i < n ? (len + UNIT - 1) / UNIT : 0;
            if (i < n) { kstart[i] = st4[u]; klen[i] = len; }
            int x = nu;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) { int y = __shfl_up_sync(0xffffffffu, x, o); if (lane >= o) x += y; }
            if (i < n) ucum[i] = carry + x - nu;
            carry += __shfl_sync(0xffffffffu, x, 31);
          }
        }
        if (lane == 0) { ucum[n] = carry; meta[0] = carry; meta[1] = n; }
        __syncwarp();
        if (lane == 0) mbar_arrive(tab_full + tb);
        // Q tiles of this item, once the last QK of the previous item has read the Q buffer
        if (lane == 0) {
          if (li >= 1) mbar_wait(q_empty, (li - 1) & 1);
          const int ntq = it.has1 ? 2 : 1;
          mbar_arrive_expect_tx(q_full, ntq * L::QT);
          for (int tq = 0; tq < ntq; ++tq)
            for (int hf = 0; hf < L::HALVES; ++hf)
              tma_load_2d(sm + L::OFF_Q + tq * L::QT + hf * L::HALF_Q, &tm_q, hf * 64,
                          bh * N + it.qbeg + (it.t0 + tq) * BM, q_full);
        }
        __syncwarp();
      } else {
        mbar_wait(tab_full + tb, (li >> 1) & 1);
      }
      const int U = meta[0], nkeep = meta[1];
      const int nt = (U + UPT - 1) / UPT;
      int cur = 0;
      auto unit_row = [&](int jj) -> int {
        const int g = jj * UPT + lane;
        while (cur + 1 < nkeep && ucum[cur + 1] <= jj * UPT) ++cur;
        int i = cur, row = bh * N + kstart[0];
        if (lane < UPT && g < U) {
          while (i + 1 < nkeep && ucum[i + 1] <= g) ++i;
          row = bh * N + kstart[i] + (g - ucum[i]) * UNIT;
        }
        return row;
      };
      for (int jj = 0; jj < nt; ++jj) {
        const int s = jj % NST;
        const int row = unit_row(jj);
        mbar_wait(empty + s, (use[s] & 1) ^ 1);
        ++use[s];
        uint8_t* base = ring + s * L::KT;
        const int prev = __shfl_up_sync(0xffffffffu, row, 1);
        const bool start = lane < UPT && (lane == 0 || row != prev + UNIT);
        const uint32_t starts = __ballot_sync(0xffffffffu, start) | (1u << UPT);
        if (lane == 0) mbar_arrive_expect_tx(full + s, L::KT);
        __syncwarp();
        if (start) {
          const uint32_t after = starts & ~((2u << lane) - 1u);
          const int len = __ffs(after) - 1 - lane;
          int off = 0;
#pragma unroll
          for (int bi = 4; bi >= 0; --bi) {
            if (len & (1 << bi)) {
              const CUtensorMap* m = is_v ? &kv.v[bi] : &kv.k[bi];
#pragma unroll
              for (int hf = 0; hf < L::HALVES; ++hf)
                tma_load_2d(base + hf * L::HALF_K + (lane + off) * 1024, m, hf * 64, row + off * UNIT, full + s);
              off += 1 << bi;
            }
          }
        }
        __syncwarp();
      }
      if (is_v && lane == 0) mbar_arrive(tab_free + tb);
    }
  } else if (warp == WARP_MMA) {
    // ================= MMA issuer =================
    constexpr uint32_t idesc_qk = idesc_bf16(BM, BN, 0, 0);
    constexpr uint32_t idesc_pv = idesc_bf16(BM, D, 0, 1);
    const uint64_t dq0 = smem_desc_sw128(smem_u32(sm + L::OFF_Q), 16, 1024);
    const uint64_t dk0 = smem_desc_sw128(smem_u32(sm + L::OFF_K), 16, 1024);
    const uint64_t dv0 = smem_desc_sw128(smem_u32(sm + L::OFF_V), L::HALF_K, 1024);
    int ku[2] = {0, 0}, vu[2] = {0, 0}, pc[2] = {0, 0};
    auto issue_qk = [&](int tq, int s, int qs) {
      if (elect_one()) {
        const uint32_t d_tmem = tmem + tq * 128;
        const uint64_t qd = dq0 + (uint64_t)((qs * L::QT) >> 4);
        const uint64_t kd = dk0 + (uint64_t)((s * L::KT) >> 4);
#pragma unroll
        for (int kk2 = 0; kk2 < D / 16; ++kk2) {
          const uint32_t off = ((kk2 >> 2) * L::HALF_Q + (kk2 & 3) * 32) >> 4;
          const uint32_t offk = ((kk2 >> 2) * L::HALF_K + (kk2 & 3) * 32) >> 4;
          mma_ss(d_tmem, qd + off, kd + offk, idesc_qk, kk2 > 0);
        }
      }
      __syncwarp();
    };
    auto issue_pv = [&](int tq, int s, int half, bool acc) {
      if (elect_one()) {
        const uint32_t d_tmem = tmem + 256 + tq * 128;
        const uint32_t p_tmem = tmem + tq * 128;
        const uint64_t vd = dv0 + (uint64_t)((s * L::KT) >> 4);
#pragma unroll
        for (int k4 = 0; k4 < BN / 32; ++k4) {
          const int kk2 = half * (BN / 32) + k4;
          mma_ts(d_tmem, p_tmem + kk2 * 8, vd + (uint64_t)((kk2 * 2048) >> 4), idesc_pv, (acc || kk2 > 0) ? 1u : 0u);
        }
      }
      __syncwarp();
    };
    auto commit = [&](uint64_t* bar) {
      if (elect_one()) mma_commit(bar);
      __syncwarp();
    };
    auto wait_k = [&](int s) { mbar_wait(k_full + s, ku[s] & 1); ++ku[s]; tc_fence_after(); };
    auto wait_v = [&](int s) { mbar_wait(v_full + s, vu[s] & 1); ++vu[s]; };
    for (int li = 0; next_item(slot, total_slots, items_ub, kq, item_start, offs_q, it); ++li) {
      const int tb = li & 1;
      mbar_wait(tab_full + tb, (li >> 1) & 1);
      const int nt = (tab_meta(tb)[0] + UPT - 1) / UPT;
      __syncwarp();
      if (lane == 0) mbar_arrive(tab_free + tb);
      bool first_pv = true;
      // PV of set tq on V slot s (item-local KV index j decides accumulate); the first PV of an item
      // overwrites O, so it waits until the previous item's epilogue has read O
      auto wait_pv = [&](int tq, int s, int j) {
        if (first_pv) {
          if (li >= 1) mbar_wait(o_free, (li - 1) & 1);
          first_pv = false;
        }
        const int par = pc[tq] & 1;
        ++pc[tq];
        mbar_wait(p_full + tq * 2 + 0, par);
        tc_fence_after();
        issue_pv(tq, s, 0, j > 0);
        mbar_wait(p_full + tq * 2 + 1, par);
        tc_fence_after();
        issue_pv(tq, s, 1, true);
      };
      mbar_wait(q_full, li & 1);
      if (!it.split) {
        wait_k(0);
        issue_qk(0, 0, 0);
        commit(s_full + 0);
        issue_qk(1, 0, 1);
        commit(s_full + 1);
        commit(k_empty + 0);
        if (nt == 1) commit(q_empty);
        for (int j = 0; j < nt; ++j) {
          const int s = j % NST, s1 = (j + 1) % NST;
          const bool more = j + 1 < nt;
          wait_v(s);
          wait_pv(0, s, j);
          if (more) {
            wait_k(s1);
            issue_qk(0, s1, 0);
            commit(s_full + 0);
          }
          wait_pv(1, s, j);
          commit(v_empty + s);
          if (more) {
            issue_qk(1, s1, 1);
            commit(s_full + 1);
            commit(k_empty + s1);
            if (j + 2 == nt) commit(q_empty);  // the item's last QK is issued
          }
        }
      } else {
        wait_k(0);
        issue_qk(0, 0, 0);
        commit(s_full + 0);
        commit(k_empty + 0);
        if (nt > 1) {
          wait_k(1);
          issue_qk(1, 1, 0);
          commit(s_full + 1);
          commit(k_empty + 1);
        }
        if (nt <= 2) commit(q_empty);
        for (int j = 0; 2 * j < nt; ++j) {
          const bool has_b = 2 * j + 1 < nt, more_a = 2 * j + 2 < nt, more_b = 2 * j + 3 < nt;
          wait_v(0);
          wait_pv(0, 0, j);
          commit(v_empty + 0);
          if (more_a) {
            wait_k(0);
            issue_qk(0, 0, 0);
            commit(s_full + 0);
            commit(k_empty + 0);
            if (2 * j + 3 >= nt) commit(q_empty);  // tile 2j+2 is the last
          }
          if (has_b) {
            wait_v(1);
            wait_pv(1, 1, j);
            commit(v_empty + 1);
            if (more_b) {
              wait_k(1);
              issue_qk(1, 1, 0);
              commit(s_full + 1);
              commit(k_empty + 1);
              if (2 * j + 4 >= nt) commit(q_empty);  // tile 2j+3 is the last
            }
          }
        }
      }
      commit(o_full);
    }
  } else {
    // ================= softmax / epilogue (warps 0-7) =================
    const int tq = warp >> 2;
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const uint32_t s_tm = tmem + lane_off + tq * 128;
    const uint32_t o_tm = tmem + lane_off + 256 + tq * 128;
    int sc = 0;  // S tiles of this set consumed (s_full parity), across items
    for (int li = 0; next_item(slot, total_slots, items_ub, kq, item_start, offs_q, it); ++li) {
      const int tb = li & 1;
      mbar_wait(tab_full + tb, (li >> 1) & 1);
      const int* klen = tab_klen(tb);
      const int* ucum = tab_ucum(tb);
      const int U = tab_meta(tb)[0], nkeep = tab_meta(tb)[1];
      const int nt = (U + UPT - 1) / UPT;
      const bool split = it.split;
      const int my_nt = split ? (nt + 1 - tq) / 2 : nt;
      float m = -INFINITY, l = 0.f;
      int ci = 0;
      uint32_t mw0 = 0, mw1 = 0, mw2 = 0, mw3 = 0;
      auto tile_mask = [&](int j) {
        mw0 = mw1 = mw2 = mw3 = 0;
        const int g0 = j * UPT;
        while (ci < nkeep) {
          const int gl = ucum[ci + 1] - 1;
          if (gl >= g0 + UPT) break;
          const int vc = klen[ci] - UNIT * (gl - ucum[ci]);
          if (vc < UNIT && gl >= ucum[ci] && gl >= g0) {
            const int u = gl - g0;
            const uint32_t bits = ((0xffu << vc) & 0xffu) << (8 * (u & 3));
            const int w = u >> 2;
            mw0 |= w == 0 ? bits : 0u; mw1 |= w == 1 ? bits : 0u;
            mw2 |= w == 2 ? bits : 0u; mw3 |= w == 3 ? bits : 0u;
          }
          ++ci;
        }
        if (g0 + UPT > U) {
          for (int u = U - g0; u < UPT; ++u) {
            const uint32_t bits = 0xffu << (8 * (u & 3));
            const int w = u >> 2;
            mw0 |= w == 0 ? bits : 0u; mw1 |= w == 1 ? bits : 0u;
            mw2 |= w == 2 ? bits : 0u; mw3 |= w == 3 ? bits : 0u;
          }
        }
      };
      if (my_nt > 0) tile_mask(split ? tq : 0);
      for (int j = 0; j < my_nt; ++j) {
        mbar_wait(s_full + tq, sc & 1);
        ++sc;
        tc_fence_after();
        uint32_t su[BN];
#pragma unroll
        for (int c = 0; c < BN / 32; ++c) tmem_ld32(s_tm + c * 32, su + c * 32);
        tmem_wait_ld();
#define CS_APPLY_MASK(W, MWV)                                                        \
  if (MWV) {                                                                         \
    _Pragma("unroll") for (int r2 = 0; r2 < 32; ++r2) if ((MWV >> r2) & 1u) su[W * 32 + r2] = 0xff800000u; \
  }
        CS_APPLY_MASK(0, mw0)
        CS_APPLY_MASK(1, mw1)
        CS_APPLY_MASK(2, mw2)
        CS_APPLY_MASK(3, mw3)
#undef CS_APPLY_MASK
        float mx8[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) mx8[i] = fmaxf(__uint_as_float(su[i]), __uint_as_float(su[8 + i]));
#pragma unroll
        for (int c = 16; c < BN; c += 16)
#pragma unroll
          for (int i = 0; i < 8; ++i) mx8[i] = fmax3(mx8[i], __uint_as_float(su[c + i]), __uint_as_float(su[c + 8 + i]));
        const float mx = fmax3(fmax3(mx8[0], mx8[1], mx8[2]), fmax3(mx8[3], mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])) *
                         scale_log2;
        float alpha = 1.f;
        if (j == 0) {
          m = mx;
        } else if (mx > m + kRescaleThresh) {
          alpha = ex2(m - mx);
          l *= alpha;
          m = mx;
        }
        const bool warp_rescale = __any_sync(0xffffffffu, alpha != 1.f);
        const float2 sl2 = make_float2(scale_log2, scale_log2), nm2 = make_float2(-m, -m);
        float2 acc4[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
#pragma unroll
          for (int c = hf * (BN / 2); c < (hf + 1) * (BN / 2); c += 2) {
            const float2 x = ffma2(make_float2(__uint_as_float(su[c]), __uint_as_float(su[c + 1])), sl2, nm2);
            const float2 p = (kPolyEvery > 0 && ((c >> 1) % kPolyEvery) == kPolyEvery - 1)
                                 ? ex2_poly2(x) : make_float2(ex2(x.x), ex2(x.y));
            acc4[(c >> 1) & 3] = fadd2(acc4[(c >> 1) & 3], p);
            su[c >> 1] = pack_bf16x2(p.x, p.y);
          }
          tmem_st32(s_tm + hf * 32, su + hf * 32);
          if (hf == 0 && warp_rescale) {
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
          mbar_arrive(p_full + tq * 2 + hf);
        }
        const float2 s01 = fadd2(acc4[0], acc4[1]), s23 = fadd2(acc4[2], acc4[3]);
        const float2 s4 = fadd2(s01, s23);
        l += s4.x + s4.y;
        if (j + 1 < my_nt) tile_mask(split ? 2 * (j + 1) + tq : j + 1);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(tab_free + tb);  // this warp is done with the item's table
      // ---- epilogue (every softmax thread waits for the item's last MMA, so a set that had no
      // tiles cannot run a whole item ahead on o_free)
      mbar_wait(o_full, li & 1);
      tc_fence_after();
      if (my_nt > 0) {
        const int prow = (it.t0 + (split ? 0 : tq)) * BM + r;
        const bool row_ok = prow < it.qlen;
        const int bh = it.bh;
        const int tok = row_ok ? perm_q[(size_t)bh * N + it.qbeg + prow] : 0;
        const int b = bh / H, h = bh % H;
        __nv_bfloat16* dst;
        if (peer_ptrs) {
          const int pr = tok / peer_npr;
          dst = reinterpret_cast<__nv_bfloat16*>(peer_ptrs[pr]) + (long long)(tok - pr * peer_npr) * osn +
                (long long)(peer_head_base + h) * osh;
        } else {
          dst = out + (long long)b * osb + (long long)h * osh + (long long)tok * osn;
        }
        if (split && nt > 1) {
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
          // xch is rewritten by the next split item only after both sets pass that item's tiles
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
      tc_fence_before();
      mbar_arrive(o_free);  // O of this item has been read (the next item's first PV may overwrite it)
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == WARP_MMA) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

}  // namespace attn_p

cudaError_t launch_bsa_fwd_persist(const CUtensorMap* tm_q, const KVMaps* kv, int BH, int H, int N, int d, int kq,
                                   int kk, const int32_t* perm_q, const int32_t* offs_q, const int32_t* offs_k,
                                   const int32_t* n_keep, const int32_t* n_rows, const int32_t* kept,
                                   const int32_t* item_start, int items_ub, float scale, __nv_bfloat16* o,
                                   long long osb, long long osh, long long osn, const uint64_t* peer_ptrs,
                                   int peer_npr, int peer_head_base, cudaStream_t st) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int total_slots = BH * items_ub;
  const int grid = total_slots < sms ? total_slots : sms;
  const float scale_log2 = scale * 1.4426950408889634f;
  auto run = [&](auto kfn, int smem) -> cudaError_t {
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    kfn<<<grid, attn_p::NTHREADS, smem, st>>>(*tm_q, *kv, H, N, kq, kk, perm_q, offs_q, offs_k, n_keep, n_rows, kept,
                                              item_start, items_ub, total_slots, scale_log2, o, osb, osh, osn,
                                              peer_ptrs, peer_npr, peer_head_base);
    return cudaGetLastError();
  };
  return d == 128 ? run(attn_p::k_bsa_fwd_persist<128>, attn_p::Smem<128>::ALLOC)
                  : run(attn_p::k_bsa_fwd_persist<64>, attn_p::Smem<64>::ALLOC);
}

}  // namespace cs
