// Microtest: TMA tile::gather4 on sm_100a.  2D bf16 tensor [rows, 128] (value = row*1000+col),
// box {64, 1} SWIZZLE_128B; gather rows {r0..r3} (two 64-column halves) into a 1024-aligned SMEM
// buffer and dump it raw, so the host can check placement and the 128B swizzle.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include "../../paper_2603_18636_b200/csrc/common.cuh"
using namespace cs;

__global__ void g4(const __grid_constant__ CUtensorMap tm, int r0, int r1, int r2, int r3, int off, uint16_t* out) {
  __shared__ __align__(1024) uint8_t buf[2048];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
    mbar_arrive_expect_tx(&bar, 2 * 4 * 128);
    for (int hf = 0; hf < 2; ++hf)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(buf + hf * 1024 + off)),
          "l"(&tm), "r"(hf * 64), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(&bar))
          : "memory");
    mbar_wait(&bar, 0);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) out[i] = reinterpret_cast<uint16_t*>(buf)[i];
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  const int R = 1000, C = 128;
  std::vector<uint16_t> h(R * C);
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < C; ++c) { __nv_bfloat16 b = __float2bfloat16((float)((r % 200) * 10 + (c % 8))); h[r * C + c] = *reinterpret_cast<uint16_t*>(&b); }
  uint16_t *d, *o;
  cudaMalloc(&d, h.size() * 2); cudaMalloc(&o, 1024 * 2);
  cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  void* fp; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  Enc enc = (Enc)fp;
  for (int boxh : {1})
  for (int off : {0, 512}) {
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)R}, strides[1] = {(cuuint64_t)C * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)boxh}, es[2] = {1, 1};
    CUresult rr = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("boxh=%d encode rc=%d\n", boxh, (int)rr);
    if (rr) continue;
    cudaMemset(o, 0, 2048);
    g4<<<1, 128>>>(tm, 5, 900, 17, 3, off, o);
    cudaError_t e = cudaDeviceSynchronize();
    printf("  launch: %s\n", cudaGetErrorString(e));
    if (e) return 1;
    std::vector<uint16_t> hb(1024);
    cudaMemcpy(hb.data(), o, 2048, cudaMemcpyDeviceToHost);
    // expected: half hf, row k (0..3) of rows {5,900,17,3}, 16-byte chunk j of the 128-byte row at
    // position (j ^ k) (SWIZZLE_128B: chunk index XOR row index within the 8-row atom)
    int rows[4] = {5, 900, 17, 3}, bad = 0;
    for (int hf = 0; hf < 2; ++hf)
      for (int k = 0; k < 4; ++k)
        for (int j = 0; j < 8; ++j)
          for (int e8 = 0; e8 < 8; ++e8) {
            const int col = hf * 64 + j * 8 + e8;
            const uint16_t want = h[rows[k] * C + col];
            const int kr = k + off / 128;  // row within the 8-row swizzle atom
            const uint16_t got = hb[hf * 512 + kr * 64 + ((j ^ kr) * 8) + e8];
            if (want != got) ++bad;
          }
    printf("  dst offset %d: swizzled-placement mismatches: %d of 512\n", off, bad);
  }
  return 0;
}
