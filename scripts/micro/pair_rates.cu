// Microbenchmark: tcgen05.mma issue rate with cta_group::2 (a 2-SM pair, M = 256: each SM computes
// its 128 rows) against cta_group::1 (M = 128), for the attention's two forms at N = 128, K = 16:
// SS (A and B from SMEM: QK^T; per SM 4 KB of A and, paired, 2 KB of B per instruction) and TS
// (A from TMEM, B MN-major from SMEM: PV).  Two accumulators interleaved K-step by K-step (the
// single-CTA micro, mma_shapes.cu, shows one accumulator is latency-bound).  Prints cycles per
// instruction (per SM: the pair instruction does each SM's 128-row share in that time).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 pair_rates.cu -o pair_rates
#include <cstdio>
#include "../../paper_2603_18636_b200/csrc/common.cuh"
using namespace cs;

CS_DEV void mma_ts_pair(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(acc)
      : "memory");
}

template <bool PAIR>
__global__ void __launch_bounds__(128, 1) k(long long* out, int iters, int mode) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = PAIR ? cluster_ctarank() : 0;
  for (int i = threadIdx.x; i < 131072 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  fence_proxy_async_smem();
  if constexpr (PAIR) cluster_sync_all();
  if (warp == 0) {
    if constexpr (PAIR) tmem_alloc_pair(&slot, 512); else tmem_alloc(&slot, 512);
  }
  tc_fence_before();
  if constexpr (PAIR) cluster_sync_all(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 0 && rank == 0) {
    const uint32_t sa = smem_u32(sm), sb = smem_u32(sm + 65536);
    const uint32_t id_ss = idesc_bf16(PAIR ? 256 : 128, 128, 0, 0), id_ts = idesc_bf16(PAIR ? 256 : 128, 128, 0, 1);
    const uint64_t ad0 = smem_desc_sw128(sa, 16, 1024), bd0 = smem_desc_sw128(sb, 16, 1024);
    const uint64_t vd0 = smem_desc_sw128(sb, 64 * 128, 1024);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = ((kk >> 2) * 16384 + (kk & 3) * 32) >> 4;
          const uint64_t vo = (uint64_t)((kk * 2048) >> 4);
          if (mode == 0) {
            if constexpr (PAIR) {
              mma_ss_pair(tmem, ad0 + off, bd0 + off, id_ss, 1);
              mma_ss_pair(tmem + 128, ad0 + off, bd0 + off, id_ss, 1);
            } else {
              mma_ss(tmem, ad0 + off, bd0 + off, id_ss, 1);
              mma_ss(tmem + 128, ad0 + off, bd0 + off, id_ss, 1);
            }
          } else {
            if constexpr (PAIR) {
              mma_ts_pair(tmem + 256, tmem + kk * 8, vd0 + vo, id_ts, 1);
              mma_ts_pair(tmem + 384, tmem + 128 + kk * 8, vd0 + vo, id_ts, 1);
            } else {
              mma_ts(tmem + 256, tmem + kk * 8, vd0 + vo, id_ts, 1);
              mma_ts(tmem + 384, tmem + 128 + kk * 8, vd0 + vo, id_ts, 1);
            }
          }
        }
      }
      __syncwarp();
    }
    if constexpr (PAIR) { if (elect_one()) mma_commit_pair(&bar); }
    else { if (elect_one()) mma_commit(&bar); }
    __syncwarp();
    mbar_wait(&bar, 0);
    if (threadIdx.x == 0) out[0] = clock64() - t0;
  }
  if constexpr (PAIR) {
    if (warp == 0 && rank == 1) mbar_wait(&bar, 0);  // the multicast commit arrives here too
  }
  tc_fence_before();
  if constexpr (PAIR) cluster_sync_all(); else __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    if constexpr (PAIR) tmem_dealloc_pair(tmem, 512); else tmem_dealloc(tmem, 512);
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(k<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 140000);
  cudaFuncSetAttribute(k<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 140000);
  const int iters = 4000;
  const char* names[] = {"SS (QK) two accs", "TS (PV) two accs"};
  for (int mode = 0; mode < 2; ++mode) {
    for (int pair = 0; pair < 2; ++pair) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(pair ? 2 : 1);
      cfg.blockDim = dim3(128);
      cfg.dynamicSmemBytes = 140000;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = pair ? 2 : 1;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      cudaError_t e = pair ? cudaLaunchKernelEx(&cfg, k<true>, d, iters, mode) : cudaLaunchKernelEx(&cfg, k<false>, d, iters, mode);
      long long h = 0;
      cudaError_t e2 = cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      printf("%-18s %s: %7.2f cycles per instruction (%s / %s)\n", names[mode], pair ? "cta_group::2 M=256" : "cta_group::1 M=128",
             (double)h / (iters * 16.0), cudaGetErrorString(e), cudaGetErrorString(e2));
    }
  }
  return 0;
}
