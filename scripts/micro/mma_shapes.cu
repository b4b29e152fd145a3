// Microbenchmark: tcgen05.mma kind::f16 issue rate (cycles per M=128, K=16 instruction) for the
// attention's two MMA forms — SS (A and B from SMEM, K-major SWIZZLE_128B: QK^T) and TS (A from
// TMEM, B MN-major from SMEM: PV) — versus N and versus how consecutive instructions share their
// accumulator: one CTA, one elected lane of a warp issuing precomputed descriptors back to back.
//   mode 0: SS, 8 K-steps into one accumulator (then the next accumulator)
//   mode 1: SS, K-steps of two accumulators interleaved (acc0 k0, acc1 k0, acc0 k1, ...)
//   mode 2: TS, 8 K-steps into one accumulator
//   mode 3: TS, two accumulators interleaved
//   mode 4: SS and TS interleaved (QK of one tile between the PV steps of the other)
//   mode 5: one attention step of BN = N keys: QK pair (SS, two accumulators interleaved, 8 K-steps)
//           then PV pair (TS N=128, two accumulators interleaved, N/16 K-steps)
//   mode 6: TS split by output columns: N=64 into O[:, 0:64] and O[:, 64:128] interleaved (one PV
//           of a 128-wide head as two independent accumulators), 8 K-steps
//   mode 7: SS at M = 64 (a half-height Q tile), K-steps of two accumulators interleaved
//   mode 8: TS at M = 64 (P of a half-height tile from TMEM), two accumulators interleaved
// ldw > 0: that many extra warps continuously tcgen05.ld their lanes' 64 S columns (the softmax
// warps' TMEM reads competing with the MMAs' accumulator traffic)
// The chain-free floor is 128 N / 256 = N / 2 cycles per instruction.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 mma_shapes.cu -o mma_shapes
#include <cstdio>
#include "../../paper_2603_18636_b200/csrc/common.cuh"
using namespace cs;

__global__ void __launch_bounds__(352, 1) k(long long* out, int iters, int n, int mode, int ldw) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  __shared__ volatile int done;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) done = 0;
  for (int i = threadIdx.x; i < 131072 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc(&slot, 512);
  fence_proxy_async_smem();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 0) {
    const uint32_t sa = smem_u32(sm), sb = smem_u32(sm + 65536);
    const uint32_t id_ss = idesc_bf16(128, n, 0, 0), id_ts = idesc_bf16(128, 128, 0, 1);
    const uint64_t ad0 = smem_desc_sw128(sa, 16, 1024), bd0 = smem_desc_sw128(sb, 16, 1024);
    const uint64_t vd0 = smem_desc_sw128(sb, 128 * 128, 1024);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = ((kk >> 2) * 16384 + (kk & 3) * 32) >> 4;
          const uint64_t vo = (uint64_t)((kk * 2048) >> 4);
          if (mode == 0) {
            mma_ss(tmem + (it & 1) * 128, ad0 + off, bd0 + off, id_ss, 1);
          } else if (mode == 1) {
            mma_ss(tmem, ad0 + off, bd0 + off, id_ss, 1);
            mma_ss(tmem + 128, ad0 + off, bd0 + off, id_ss, 1);
          } else if (mode == 2) {
            mma_ts(tmem + 256 + (it & 1) * 128, tmem + kk * 8, vd0 + vo, id_ts, 1);
          } else if (mode == 3) {
            mma_ts(tmem + 256, tmem + kk * 8, vd0 + vo, id_ts, 1);
            mma_ts(tmem + 384, tmem + 128 + kk * 8, vd0 + vo, id_ts, 1);
          } else if (mode == 6) {
            const uint32_t id64 = idesc_bf16(128, 64, 0, 1);
            mma_ts(tmem + 256, tmem + kk * 8, vd0 + vo, id64, 1);
            mma_ts(tmem + 320, tmem + kk * 8, vd0 + vo + (uint64_t)(8192 >> 4), id64, 1);
          } else if (mode == 7) {
            const uint32_t id64m = idesc_bf16(64, n, 0, 0);
            mma_ss(tmem, ad0 + off, bd0 + off, id64m, 1);
            mma_ss(tmem + 256, ad0 + off, bd0 + off, id64m, 1);
          } else if (mode == 8) {
            const uint32_t id64m = idesc_bf16(64, 128, 0, 1);
            mma_ts(tmem + 256, tmem + kk * 8, vd0 + vo, id64m, 1);
            mma_ts(tmem + 384, tmem + 128 + kk * 8, vd0 + vo, id64m, 1);
          } else if (mode == 4) {
            mma_ss(tmem, ad0 + off, bd0 + off, id_ss, 1);
            mma_ts(tmem + 256, tmem + 128 + kk * 8, vd0 + vo, id_ts, 1);
          } else {
            mma_ss(tmem, ad0 + off, bd0 + off, id_ss, 1);
            mma_ss(tmem + 128, ad0 + off, bd0 + off, id_ss, 1);
          }
        }
        if (mode == 5)
          for (int kk = 0; kk < n / 16; ++kk) {
            const uint64_t vo = (uint64_t)((kk * 2048) >> 4);
            mma_ts(tmem + 256, tmem + 80 + kk * 8, vd0 + vo, id_ts, 1);
            mma_ts(tmem + 384, tmem + 208 + kk * 8, vd0 + vo, id_ts, 1);
          }
      }
      __syncwarp();
    }
    if (elect_one()) mma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    if (threadIdx.x == 0) out[0] = clock64() - t0;
    if (threadIdx.x == 0) done = 1;
  } else if (warp >= 2 && warp < 2 + ldw) {
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    uint32_t acc = 0;
    while (!done) {
      uint32_t r[32];
      tmem_ld32(tmem + lane_off + (warp & 4 ? 128 : 0), r);
      tmem_ld32(tmem + lane_off + (warp & 4 ? 160 : 32), r);
      tmem_wait_ld();
      acc += r[0];
    }
    if (acc == 12345) out[1] = acc;
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 140000);
  const int iters = 4000;
  const char* names[] = {"SS one acc", "SS two accs interleaved", "TS(N=128) one acc", "TS(N=128) two accs",
                         "SS + TS(N=128) interleaved", "attention step (QK2 + PV2)",
                         "TS N=64 x2 (split O columns)", "SS M=64 two accs", "TS M=64 N=128 two accs"};
  for (int ldw = 0; ldw <= 8; ldw += 8)
    for (int mode = 0; mode < 9; ++mode)
      for (int n : {64, 80, 96, 128, 256}) {
        if (((mode >= 2 && mode <= 3) || mode == 6 || mode == 8) && n != 128) continue;
        if (mode == 5 && n > 128) continue;
        k<<<1, 352, 140000>>>(d, iters, n, mode, ldw);
        long long h = 0;
        cudaError_t e = cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        const int per_it = mode == 5 ? 16 + 2 * (n / 16) : ((mode == 1 || mode == 3 || mode == 4 || mode >= 6) ? 16 : 8);
        const double floor_c = mode == 5 ? (16 * n / 2 + 2 * (n / 16) * 64) / (double)per_it
                                         : (mode == 4 ? (n / 2 + 64) / 2.0 : (mode == 6 ? 32 : (mode >= 2 ? 64 : n / 2)));
        printf("ldw=%d %-28s N=%3d: %7.2f cycles per instruction (floor %.1f)%s %s\n", ldw, names[mode], n,
               (double)h / (iters * (double)per_it), floor_c,
               mode == 5 ? "" : "", cudaGetErrorString(e));
        if (mode == 5) printf("      -> %.0f cycles per attention step of %d keys (2 Q tiles)\n", (double)h / iters, n);
      }
  return 0;
}
