// Microtest: CTA-pair tcgen05 MMA (cta_group::2) on sm_100a, the building block of a 2-SM
// assignment GEMM.  One cluster of 2 CTAs computes D[256 x 256] = A[256 x 64] . B[256 x 64]^T:
// CTA r loads A rows [128r, 128r+128) and B rows [128r, 128r+128) with TMA (completion counted on
// the leader CTA's mbarrier), the leader issues 4 MMAs of M=256 N=256 K=16 and multicasts the commit
// to both CTAs; each CTA reads its 128 TMEM lanes and writes those rows of D.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 pair_mma_test.cu -o pair_mma_test -lcuda
#include <cuda.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>
#include "../../paper_2603_18636_b200/csrc/common.cuh"
using namespace cs;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa_u32(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    k_pair(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, float* D) {
  extern __shared__ uint8_t smraw[];
  uint8_t* sm = smraw + ((1024u - (smem_u32(smraw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + 32768);
  uint64_t* done = full + 1;
  uint32_t* slot = reinterpret_cast<uint32_t*>(sm + 32768 + 64);
  const uint32_t rank = cluster_rank();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(full, 1);
    mbar_init(done, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (threadIdx.x == 0) {
    const uint32_t full_leader = mapa_u32(smem_u32(full), 0);
    if (rank == 0) mbar_arrive_expect_tx(full, 4 * 16384);
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(sm)), "l"(&ta), "r"(0), "r"((int)(128 * rank)),
        "r"(full_leader)
        : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(sm + 16384)), "l"(&tb), "r"(0), "r"((int)(128 * rank)),
        "r"(full_leader)
        : "memory");
    if (rank == 0) {
      mbar_wait(full, 0);
      tc_fence_after();
      const uint32_t idesc = idesc_bf16(256, 256, 0, 0);
      for (int k = 0; k < 4; ++k) {
        const uint64_t ad = smem_desc_sw128(smem_u32(sm) + k * 32, 16, 1024);
        const uint64_t bd = smem_desc_sw128(smem_u32(sm + 16384) + k * 32, 16, 1024);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(ad), "l"(bd), "r"(idesc), "r"(k > 0 ? 1u : 0u)
            : "memory");
      }
      asm volatile(
          "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
              smem_u32(done)),
          "h"((uint16_t)3)
          : "memory");
    }
  }
  __syncwarp();
  mbar_wait(done, 0);
  tc_fence_after();
  const int row = warp * 32 + lane;
  for (int c0 = 0; c0 < 256; c0 += 16) {
    uint32_t v[16];
    tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c0, v);
    tmem_wait_ld();
    for (int i = 0; i < 16; ++i) D[(size_t)(128 * rank + row) * 256 + c0 + i] = __uint_as_float(v[i]);
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
  }
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int R = 256, K = 64;
  std::vector<uint16_t> ha(R * K), hb(R * K);
  std::vector<float> fa(R * K), fb(R * K);
  uint32_t s = 12345;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return ((s >> 9) & 0xFFFF) / 65536.0f - 0.5f; };
  for (int i = 0; i < R * K; ++i) {
    __nv_bfloat16 a = __float2bfloat16(rnd()), b = __float2bfloat16(rnd());
    ha[i] = *reinterpret_cast<uint16_t*>(&a); hb[i] = *reinterpret_cast<uint16_t*>(&b);
    fa[i] = __bfloat162float(a); fb[i] = __bfloat162float(b);
  }
  uint16_t *da, *db; float* dd;
  cudaMalloc(&da, R * K * 2); cudaMalloc(&db, R * K * 2); cudaMalloc(&dd, R * R * 4);
  cudaMemcpy(da, ha.data(), R * K * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(db, hb.data(), R * K * 2, cudaMemcpyHostToDevice);
  cudaMemset(dd, 0xff, R * R * 4);
  void* fp; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  Enc enc = (Enc)fp;
  CUtensorMap ta, tb;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)R}, strides[1] = {(cuuint64_t)K * 2};
  cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
  enc(&ta, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, da, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&tb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, db, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int smem = 32768 + 128 + 1024;
  cudaFuncSetAttribute(k_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_pair<<<2, 128, smem>>>(ta, tb, dd);
  cudaError_t e = cudaDeviceSynchronize();
  printf("launch: %s\n", cudaGetErrorString(e));
  if (e) return 1;
  std::vector<float> hd(R * R);
  cudaMemcpy(hd.data(), dd, R * R * 4, cudaMemcpyDeviceToHost);
  int bad = 0; double maxerr = 0;
  int quad_bad[2][2] = {{0, 0}, {0, 0}};
  for (int i = 0; i < R; ++i)
    for (int j = 0; j < R; ++j) {
      double ref = 0;
      for (int k = 0; k < K; ++k) ref += (double)fa[i * K + k] * fb[j * K + k];
      double err = fabs(ref - hd[i * R + j]);
      if (!(err <= 1e-3)) { ++bad; quad_bad[i / 128][j / 128]++; }
      if (err > maxerr || err != err) maxerr = err;
    }
  printf("bad=%d maxerr=%g quadrants(rows/cols halves) bad: %d %d %d %d\n", bad, maxerr, quad_bad[0][0], quad_bad[0][1],
         quad_bad[1][0], quad_bad[1][1]);
  printf("%s\n", bad ? "FAIL" : "PASS");
  return bad ? 1 : 0;
}
