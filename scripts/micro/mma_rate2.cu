// Microbenchmark 2: effect of tcgen05.commit frequency, mixed QK/PV shapes, and concurrent TMEM
// loads by other warps on the tcgen05.mma rate.
#include "../../paper_2603_18636_b200/csrc/common.cuh"
#include <cstdio>
using namespace cs;
// commit_every: commit after this many MMAs (0 = never); mix: alternate 8x SS N64 and 4x TS N128;
// ldw: number of extra warps continuously doing tcgen05.ld of 64 columns
__global__ void __launch_bounds__(320, 1) k(long long* out, int iters, int commit_every, int mix, int ldw) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar[2];
  __shared__ uint32_t slot;
  __shared__ volatile int done;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); done = 0; fence_barrier_init(); }
  if (warp == 9) tmem_alloc(&slot, 512);
  fence_proxy_async_smem();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 9) {
    if ((threadIdx.x & 31) == 0) {
      const uint32_t sa = smem_u32(sm), sb = smem_u32(sm + 32768);
      const uint32_t id64 = idesc_bf16(128, 64, 0, 0), id128 = idesc_bf16(128, 128, 0, 1);
      int cnt = 0;
      long long t0 = clock64();
      for (int it = 0; it < iters; ++it) {
        for (int k = 0; k < 8; ++k) {
          const uint64_t ad = smem_desc_sw128(sa + (k & 3) * 32 + (k >> 2) * 16384, 16, 1024);
          const uint64_t bd = smem_desc_sw128(sb + (k & 3) * 32 + (k >> 2) * 8192, 16, 1024);
          mma_ss(tmem + (it & 1) * 64, ad, bd, id64, 1);
          if (commit_every && ++cnt % commit_every == 0) mma_commit(&bar[0]);
        }
        if (mix)
          for (int k = 0; k < 4; ++k) {
            const uint64_t bd = smem_desc_sw128(sb + k * 2048, 8192, 1024);
            mma_ts(tmem + 256, tmem + 128 + k * 8, bd, id128, 1);
            if (commit_every && ++cnt % commit_every == 0) mma_commit(&bar[0]);
          }
      }
      mma_commit(&bar[1]);
      mbar_wait(&bar[1], 0);
      long long t2 = clock64();
      out[0] = t2 - t0;
      done = 1;
    }
    __syncwarp();
  } else if (warp < ldw) {
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    uint32_t acc = 0;
    while (!done) {
      uint32_t r[32];
      tmem_ld32(tmem + lane_off + 384, r);
      tmem_ld32(tmem + lane_off + 416, r);
      tmem_wait_ld();
      acc += r[0];
    }
    if (acc == 12345) out[1] = acc;
  }
  tc_fence_before(); __syncthreads();
  if (warp == 9) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}
int main() {
  long long* d; cudaMalloc(&d, 16); long long h[2];
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024);
  const int iters = 1000;
  struct { int ce, mix, ldw; const char* name; } cfg[] = {
      {0, 0, 0, "SS N64 only, no commit"}, {8, 0, 0, "SS N64, commit/8"}, {2, 0, 0, "SS N64, commit/2"},
      {0, 1, 0, "8x SS N64 + 4x TS N128, no commit"}, {6, 1, 0, "mixed, commit/6"},
      {0, 1, 8, "mixed + 8 warps tcgen05.ld"}, {6, 1, 8, "mixed, commit/6, + 8 ld warps"}};
  for (auto& c : cfg) {
    k<<<1, 320, 66 * 1024>>>(d, 10, c.ce, c.mix, c.ldw);
    k<<<1, 320, 66 * 1024>>>(d, iters, c.ce, c.mix, c.ldw);
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    const double ideal = iters * (8 * 32.0 + (c.mix ? 4 * 64.0 : 0));
    printf("%-40s %.0f cycles, ideal %.0f -> %.0f%%  (%s)\n", c.name, (double)h[0], ideal, 100 * ideal / h[0],
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
