// Microtest: TMA tile-mode boxes of 1..128 rows x 64 bf16 columns (SWIZZLE_128B) written to a
// 128-byte aligned (not 1024-byte aligned) shared-memory row offset.  Checks that the rows land
// exactly where a 128-row box load at the tile base would put them (chunk j of tile row R at
// 16-byte position j ^ (R & 7)), i.e. that a K/V tile can be packed from row-exact boxes.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include "../../paper_2603_18636_b200/csrc/common.cuh"
using namespace cs;

struct Maps { CUtensorMap m[8]; };

// load rows [src, src + h) of the tensor into tile rows [dst, dst + h) with the box of height h
__global__ void k(const __grid_constant__ Maps maps, int src, int dst, int h, uint16_t* out) {
  __shared__ __align__(1024) uint8_t buf[128 * 128];
  __shared__ uint64_t bar;
  for (int i = threadIdx.x; i < 128 * 128 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(buf)[i] = 0xffffffffu;
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(&bar, h * 128);
    int off = 0;
    for (int bi = 7; bi >= 0; --bi)
      if (h & (1 << bi)) {
        tma_load_2d(buf + (dst + off) * 128, &maps.m[bi], 0, src + off, &bar);
        off += 1 << bi;
      }
    mbar_wait(&bar, 0);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 128 * 64; i += blockDim.x) out[i] = reinterpret_cast<uint16_t*>(buf)[i];
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  const int R = 4096, C = 64;
  std::vector<uint16_t> h(R * C);
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < C; ++c) h[r * C + c] = (uint16_t)((r * 64 + c) & 0x7fff);
  uint16_t *d, *o;
  cudaMalloc(&d, h.size() * 2); cudaMalloc(&o, 128 * 64 * 2);
  cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  void* fp; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  Enc enc = (Enc)fp;
  Maps maps;
  for (int bi = 0; bi < 8; ++bi) {
    cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)R}, strides[1] = {(cuuint64_t)C * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)(1 << bi)}, es[2] = {1, 1};
    CUresult rr = enc(&maps.m[bi], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, strides, box, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (rr) { printf("encode box %d rc=%d\n", 1 << bi, (int)rr); return 1; }
  }
  int total_bad = 0, cases = 0;
  const int hs[] = {1, 2, 3, 5, 7, 8, 9, 13, 31, 64, 77, 100, 127, 128};
  for (int hh : hs)
    for (int dst = 0; dst + hh <= 128; dst += (hh > 60 ? 1 : 3)) {
      const int src = 1000 + 7 * dst + hh;
      k<<<1, 256>>>(maps, src, dst, hh, o);
      cudaError_t e = cudaDeviceSynchronize();
      if (e) { printf("launch (h=%d dst=%d): %s\n", hh, dst, cudaGetErrorString(e)); return 1; }
      std::vector<uint16_t> hb(128 * 64);
      cudaMemcpy(hb.data(), o, hb.size() * 2, cudaMemcpyDeviceToHost);
      int bad = 0;
      for (int k2 = 0; k2 < hh; ++k2) {
        const int tr = dst + k2;  // tile row
        for (int j = 0; j < 8; ++j)
          for (int e8 = 0; e8 < 8; ++e8)
            if (hb[tr * 64 + ((j ^ (tr & 7)) * 8) + e8] != h[(src + k2) * C + j * 8 + e8]) ++bad;
      }
      // rows outside [dst, dst + hh) untouched
      for (int tr = 0; tr < 128; ++tr)
        if (tr < dst || tr >= dst + hh)
          for (int c = 0; c < 64; ++c) if (hb[tr * 64 + c] != 0xffff) ++bad;
      total_bad += bad;
      ++cases;
      if (bad && total_bad < 2000) printf("h=%d dst=%d: %d mismatches\n", hh, dst, bad);
    }
  printf("row-exact TMA boxes: %d cases, %d mismatches\n", cases, total_bad);
  return total_bad != 0;
}
