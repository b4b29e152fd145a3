// Microtest: tcgen05.mma kind::f16 with f16 A/B and an F16 accumulator (idesc D format 0) on
// sm_100a — (1) where the 16-bit D elements land in TMEM (packed two per 32-bit column or one per
// column), (2) the issue rate against the F32-accumulator form, two accumulators interleaved.
// A[i][k] = 1, B[j][k] = (j % 8) + 1 (K = 16): D[i][j] = 16 ((j % 8) + 1).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 f16acc_test.cu -o f16acc_test
#include <cuda_fp16.h>
#include <cstdio>
#include "../../paper_2603_18636_b200/csrc/common.cuh"
using namespace cs;

__host__ __device__ constexpr uint32_t idesc_f16in(int M, int N, int dfmt) {
  return ((uint32_t)dfmt << 4)            // D format: 0 = F16, 1 = F32
         | (0u << 7) | (0u << 10)         // A, B format: F16
         | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__global__ void __launch_bounds__(128, 1) k(uint32_t* out, long long* cyc, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // A: 128 rows x 64 halves (one SW128 atom column), K-major; B: 128 rows likewise.  With
  // SWIZZLE_128B the 16-byte chunks of row r are XOR-permuted by (r & 7); constant rows do not care
  // for A, and for B every element of row j holds the same value.
  __half* A = reinterpret_cast<__half*>(sm);
  __half* B = reinterpret_cast<__half*>(sm + 16384);
  for (int i = threadIdx.x; i < 128 * 64; i += blockDim.x) {
    A[i] = __float2half(1.0f);
    B[i] = __float2half((float)((i / 64) % 8 + 1));
  }
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc(&slot, 512);
  fence_proxy_async_smem();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = slot;
  const uint64_t ad = smem_desc_sw128(smem_u32(A), 16, 1024), bd = smem_desc_sw128(smem_u32(B), 16, 1024);
  if (warp == 0) {
    if (elect_one()) {
      // poison the first 256 columns with a marker, then one MMA into column 0 (F16 D)
      mma_ss(tmem, ad, bd, idesc_f16in(128, 128, 0), 0);
      mma_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  {
    uint32_t r[32];
    tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16), r);
    tmem_wait_ld();
    if (lane == 0 && warp == 0)
      for (int c = 0; c < 32; ++c) out[c] = r[c];
    tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + 64, r);
    tmem_wait_ld();
    if (lane == 0 && warp == 0)
      for (int c = 0; c < 32; ++c) out[32 + c] = r[c];
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  // rates: 8 K-steps x two accumulators interleaved, F16 vs F32 D
  if (warp == 0) {
    for (int fmt = 0; fmt < 2; ++fmt) {
      const uint32_t id = idesc_f16in(128, 128, fmt);
      long long t0 = clock64();
      for (int it = 0; it < iters; ++it) {
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint32_t off = ((kk & 3) * 32) >> 4;
            mma_ss(tmem, ad + off, bd + off, id, 1);
            mma_ss(tmem + 256, ad + off, bd + off, id, 1);
          }
        }
        __syncwarp();
      }
      if (elect_one()) mma_commit(&bar);
      __syncwarp();
      mbar_wait(&bar, (fmt + 1) & 1);
      if (lane == 0) cyc[fmt] = clock64() - t0;
    }
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

int main() {
  uint32_t* d;
  long long* c;
  cudaMalloc(&d, 64 * 4);
  cudaMalloc(&c, 16);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  const int iters = 2000;
  k<<<1, 128, 40000>>>(d, c, iters);
  cudaError_t e = cudaDeviceSynchronize();
  uint32_t h[64];
  long long hc[2];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  cudaMemcpy(hc, c, sizeof(hc), cudaMemcpyDeviceToHost);
  printf("launch: %s\n", cudaGetErrorString(e));
  printf("row 0, TMEM columns 0..7 (raw 32-bit; as two halves):\n");
  for (int i = 0; i < 8; ++i) {
    __half_raw lo, hi;
    lo.x = (unsigned short)(h[i] & 0xffff);
    hi.x = (unsigned short)(h[i] >> 16);
    printf("  col %2d: 0x%08x  lo %.1f hi %.1f  as f32 %.1f\n", i, h[i], __half2float(__half(lo)),
           __half2float(__half(hi)), *reinterpret_cast<float*>(&h[i]));
  }
  printf("  col 64: 0x%08x\n", h[32]);
  printf("expected D[0][j] = 16 * ((j %% 8) + 1): 16, 32, 48, ...\n");
  printf("two accumulators interleaved, N=128: F16 D %.2f, F32 D %.2f cycles per instruction\n",
         hc[0] / (iters * 16.0), hc[1] / (iters * 16.0));
  return 0;
}
