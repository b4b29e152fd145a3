// Microbenchmark 3: what makes tcgen05.commit expensive?
#include "../../paper_2603_18636_b200/csrc/common.cuh"
#include <cstdio>
using namespace cs;
__global__ void __launch_bounds__(128, 1) k(long long* out, int iters, int mode) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar[4];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); mbar_init(&bar[2], 1 << 20); mbar_init(&bar[3], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&slot, 512);
  fence_proxy_async_smem();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t sa = smem_u32(sm), sb = smem_u32(sm + 32768);
    const uint32_t id = (mode >= 7) ? idesc_bf16(128, 64, 0, 0) : idesc_bf16(128, 128, 0, 0);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      for (int k = 0; k < 8; ++k) {
        const uint64_t ad = smem_desc_sw128(sa + (k & 3) * 32 + (k >> 2) * 16384, 16, 1024);
        const uint64_t bd = smem_desc_sw128(sb + (k & 3) * 32 + (k >> 2) * 8192, 16, 1024);
        mma_ss(tmem + (mode == 5 || mode == 6 ? 0 : (it & 1) * 128), ad, bd, id, mode == 5 ? 1 : (k > 0));
      }
      if (mode == 1 || mode == 8) mma_commit(&bar[0]);  // completes a phase each time
      if (mode == 2) mma_commit(&bar[2]);              // never completes
      if (mode == 3) mma_commit(&bar[it & 1]);         // alternate
      if (mode == 4) { mma_commit(&bar[0]); mbar_wait(&bar[0], it & 1); }  // synchronous
    }
    long long t1 = clock64();
    mma_commit(&bar[3]);
    mbar_wait(&bar[3], 0);
    long long t2 = clock64();
    out[0] = t1 - t0; out[1] = t2 - t0;
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}
int main() {
  long long* d; cudaMalloc(&d, 16); long long h[2];
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024);
  const char* names[] = {"no commit", "commit each 8 (phase completes)", "commit each 8 (count 2^20)",
                         "commit each 8 alternating 2 barriers", "commit + wait each 8", "same D, always accumulate", "same D, overwrite first", "N64 no commit", "N64 commit each 8"};
  for (int iters : {1000}) for (int m = 0; m < 9; ++m) {
    k<<<1, 128, 66 * 1024>>>(d, 10, m);
    k<<<1, 128, 66 * 1024>>>(d, iters, m);
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("iters %4d %-40s issue %8lld total %8lld cycles -> %.1f cyc per 8-MMA group (ideal 512)  %s\n", iters, names[m],
           h[0], h[1], (double)h[1] / iters, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
