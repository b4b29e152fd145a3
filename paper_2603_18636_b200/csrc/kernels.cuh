// kernels.cuh — declarations shared by the libcoclust translation units.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "common.cuh"

namespace cs {

constexpr int kSortTile = 1024;  // tokens per counting-sort tile
constexpr int kMaxClusters = 1024;
constexpr int kGammaRows = 64;   // anchor rows per partial Gamma (k_gamma split over C_a rows)

// Strided bf16 [B, H, N, d] view (d contiguous).
struct XView {
  const __nv_bfloat16* p;
  long long sb, sh, sn;
  int H;
  __device__ __forceinline__ const __nv_bfloat16* row(int b, int h, int n) const {
    return p + (long long)b * sb + (long long)h * sh + (long long)n * sn;
  }
};

// ---- cluster.cu
cudaError_t launch_init_sample(XView q, XView k, int BH, int N, int d, int kq, int kk,
                               unsigned long long seed, int h_off, int h_tot, const int32_t* init_q,
                               const int32_t* init_k, float* cq, float* ck, cudaStream_t st);
cudaError_t launch_anchor_prep(const float* ca, int ka, const float* cself, int ks, int ks_pad,
                               int BH, int d, void* gamma_ws /*fp64-sized scratch*/, __nv_bfloat16* wsplit,
                               cudaStream_t st);
// k-means baseline (NEXT-2): Wsplit[bh][j] = [bf16(c_j) | bf16(c_j - bf16(c_j))], bias = -||c_j||^2 / 2
cudaError_t launch_kmeans_prep(const float* cself, int ks, int ks_pad, int BH, int d, __nv_bfloat16* wsplit,
                               float* bias, cudaStream_t st);
cudaError_t launch_seg_mean(XView x, int BH, int N, int d, int K, const int32_t* perm,
                            const int32_t* offs, float* C, __nv_bfloat16* xperm, cudaStream_t st);
cudaError_t launch_csort(const int32_t* lab, int BH, int N, int K, int32_t* perm, int32_t* offs,
                         int32_t* hist, cudaStream_t st);
cudaError_t launch_block_transpose(int A, int B, size_t row_bytes, const void* src, void* dst, cudaStream_t st);
struct UlyssesSrcs {
  const uint4* p[4];
};
cudaError_t launch_ulysses_pack(int Nl, int P, int T, size_t row_bytes, size_t src_row_bytes, size_t src_off_bytes,
                                const UlyssesSrcs& srcs, void* dst, cudaStream_t st);
cudaError_t launch_permute_rows(XView x, int BH, int N, int d, const int32_t* perm,
                                __nv_bfloat16* xp, cudaStream_t st);

// ---- assign.cu : labels[bh][n] = argmax_j x_n . W_j  (tcgen05 GEMM + fused argmax epilogue)
// tm_x: 4D map over x {d, N, H, B} box {64, 128, 1, 1}; tm_w: 2D map over Wsplit {2d, BH*ks_pad}
// box {64, nch}.
int assign_chunk_n(int ks);  // centroid columns per TMEM chunk (UMMA N)
int assign_box_rows(int ks);  // W rows per TMA box (half a chunk for the CTA-pair kernel)
cudaError_t launch_assign_gemm(const CUtensorMap* tm_x, const CUtensorMap* tm_w, int B, int H, int N,
                               int d, int ks, int nch, int ks_pad, const float* bias, int32_t* labels,
                               cudaStream_t st);

// ---- select.cu
cudaError_t launch_block_select(int BH, int H, int kq, int kk, int d, const float* cq,
                                const float* ck, const int32_t* offs_q, const int32_t* offs_k,
                                const float* budget, double tau, double theta, int rule, int flags,
                                int32_t* n_keep, int32_t* n_rows, int32_t* kept, int32_t* order,
                                int32_t* cnt, double* abar, cudaStream_t st);
cudaError_t launch_worklist(int BH, int kq, const int32_t* offs_q, int32_t* item_start,
                            cudaStream_t st);
int worklist_upper_bound(int N, int kq);

// ---- attn.cu : block-sparse flash attention over cluster-sorted Q/K/V (bf16 [BH, N, d])
// K/V maps over the sorted copies, box width 64 columns, box heights kKVBoxRows[i]: 1..7 rows (a
// segment's remainder below 8) and 8 << i (i = 0..4)
constexpr int kKVBoxes = 12;
struct KVMaps {
  CUtensorMap k[kKVBoxes];
  CUtensorMap v[kKVBoxes];
};
cudaError_t launch_bsa_fwd(const CUtensorMap* tm_q, const KVMaps* kv,
                           int BH, int H, int N, int d, int kq, int kk, const int32_t* perm_q,
                           const int32_t* offs_q, const int32_t* offs_k, const int32_t* n_keep,
                           const int32_t* n_rows, const int32_t* kept, const int32_t* item_start, int items_ub,
                           float scale, __nv_bfloat16* o, long long osb, long long osh,
                           long long osn, const uint64_t* peer_ptrs, int peer_npr,
                           int peer_head_base, cudaStream_t st);

// ---- peer.cu : cross-process peer memory (CUDA IPC) and a device-side barrier over peer flags
cudaError_t launch_peer_barrier(int P, int rank, const uint64_t* peer_flags, int epoch, cudaStream_t st);

// ---- profile.cu : offline attention density (NEXT-3); tm_q / tm_k 4D maps as in assign
cudaError_t launch_attention_density(const CUtensorMap* tm_q, const CUtensorMap* tm_k, int B, int H, int N, int d,
                                     float scale, double tau, int passes, float* rs, size_t rows, int32_t* counts,
                                     double* density, cudaStream_t st);

}  // namespace cs
