// Microtest for the compute-sanitizer racecheck report on k_assign_pair:
// kernels that do NOTHING but the CTA-pair TMEM allocation protocol of k_assign_pair —
// tcgen05.alloc.cta_group::2 by one warp in each CTA of a 2-CTA cluster into a shared-memory
// slot, a cluster barrier + CTA barrier, every thread reading the slot, a cluster barrier and the
// paired dealloc — in variants that add, one at a time, what k_assign_pair does around it:
//   0 static slot, warp 0 allocates (128 threads)
//   1 + presync: a cluster barrier BEFORE the alloc
//   2 dynamic-smem slot behind 1024-byte alignment, warp 5 of 6 allocates (192 threads)
//   3 = 2 + thread 0 initialises mbarriers (fence.mbarrier_init.release.cluster) while warp 5
//       allocates (k_assign_pair's prologue)
//   4 = 3 + a cluster barrier between the mbarrier init and the alloc
// If racecheck reports hazards for some variants only, the difference names their cause.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 pair_alloc_race.cu -o pair_alloc_race
//   compute-sanitizer --tool racecheck ./pair_alloc_race <variant>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include "../../paper_2603_18636_b200/csrc/common.cuh"
using namespace cs;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) k_alloc(uint32_t* out, int presync) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (presync) cluster_sync_all();
  if (warp == 0) tmem_alloc_pair(&slot, 512);
  tc_fence_before();
  cluster_sync_all();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = slot;
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
  tc_fence_before();
  cluster_sync_all();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc_pair(t, 512);
  }
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(192, 1) k_alloc_dyn(uint32_t* out, int variant) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + 65536);
  uint32_t* slot = reinterpret_cast<uint32_t*>(sm + 65536 + 24 * 8);
  const int warp = threadIdx.x >> 5;
  if (variant >= 3 && threadIdx.x == 0) {
    for (int i = 0; i < 24; ++i) mbar_init(bars + i, 1);
    fence_barrier_init();
  }
  if (variant >= 4) cluster_sync_all();
  if (warp == 5) tmem_alloc_pair(slot, 512);
  tc_fence_before();
  cluster_sync_all();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = *slot;
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
  tc_fence_before();
  cluster_sync_all();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc_pair(t, 512);
  }
}

int main(int argc, char** argv) {
  const int variant = argc > 1 ? atoi(argv[1]) : 0;
  const int ctas = 2 * 148, nt = variant >= 2 ? 192 : 128;
  uint32_t* d;
  cudaMalloc(&d, ctas * nt * 4);
  if (variant >= 2) {
    const int smem = 65536 + 256 + 1024;
    cudaFuncSetAttribute(k_alloc_dyn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_alloc_dyn<<<ctas, nt, smem>>>(d, variant);
  } else {
    k_alloc<<<ctas, nt>>>(d, variant);
  }
  cudaError_t e = cudaDeviceSynchronize();
  uint32_t* h = (uint32_t*)malloc(ctas * nt * 4);
  cudaMemcpy(h, d, ctas * nt * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int c = 0; c < ctas; c += 2)  // both CTAs of a pair and all their threads see one address
    for (int i = 0; i < 2 * nt; ++i) bad += h[c * nt + i] != h[c * nt];
  printf("variant=%d launch=%s inconsistent=%d first=0x%x\n", variant, cudaGetErrorString(e), bad, h[0]);
  return e != cudaSuccess || bad;
}
