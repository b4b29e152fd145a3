// Microbenchmark: tcgen05.mma issue/execute rate for the shapes the attention kernel uses.
#include "../../paper_2603_18636_b200/csrc/common.cuh"
#include <cstdio>
using namespace cs;
template <int MODE, int NN = 0>  // 0: SS N=64 ; 1: SS N=128 ; 2: TS N=128 (A tmem) ; 3: SS N=256 ; 4: SS N=NN ; 5: TS N=NN (B K-major)
__global__ void __launch_bounds__(128, 1) k(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 65536 / 4; i += 128) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc(&slot, 512);
  fence_proxy_async_smem();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t sa = smem_u32(sm), sb = smem_u32(sm + 32768);
    constexpr int N = MODE >= 4 ? NN : MODE == 0 ? 64 : MODE == 3 ? 256 : 128;
    const uint32_t idesc = idesc_bf16(128, N, 0, MODE == 2 ? 1 : 0);
    constexpr bool TS = MODE == 2 || MODE == 5;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      for (int k = 0; k < 8; ++k) {
        const uint64_t ad = smem_desc_sw128(sa + (k & 3) * 32 + (k >> 2) * 16384, 16, 1024);
        const uint64_t bd = smem_desc_sw128(sb + (k & 3) * 32 + (k >> 2) * 8192, MODE == 2 ? 8192 : 16, 1024);
        if (TS) mma_ts(tmem + 256, tmem + k * 8, bd, idesc, 1);
        else mma_ss(tmem + (N > 128 ? 0 : (it & 1) * 256), ad, bd, idesc, 1);
      }
    }
    long long t1 = clock64();
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t2 = clock64();
    out[0] = t1 - t0; out[1] = t2 - t0;
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}
int main() {
  long long* d; cudaMalloc(&d, 16); long long h[2];
  const int iters = 1000;
  const char* names[] = {"SS M128 N64 K16", "SS M128 N128 K16", "TS M128 N128 K16 (A tmem, B MN-major)", "SS M128 N256 K16",
                         "SS M128 N80 K16", "SS M128 N96 K16", "TS M128 N80 K16 (B K-major)", "TS M128 N64 K16 (B K-major)", "SS M128 N112 K16"};
  void (*fns[])(long long*, int) = {k<0>, k<1>, k<2>, k<3>, k<4, 80>, k<4, 96>, k<5, 80>, k<5, 64>, k<4, 112>};
  const int Ns[] = {64, 128, 128, 256, 80, 96, 80, 64, 112};
  for (int m = 0; m < 9; ++m) {
    if (m == 3) continue;  // N=256 needs a larger B buffer
    cudaFuncSetAttribute(fns[m], cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024);
    fns[m]<<<1, 128, 66 * 1024>>>(d, 10);
    fns[m]<<<1, 128, 66 * 1024>>>(d, iters);
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    double per = (double)h[1] / (iters * 8);
    double ideal = 128.0 * Ns[m] / 256.0;
    printf("%-40s issue %.1f cyc/instr, total %.1f cyc/instr, ideal %.0f -> %.0f%% of peak  (err %s)\n", names[m],
           (double)h[0] / (iters * 8), per, ideal, 100.0 * ideal / per, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
