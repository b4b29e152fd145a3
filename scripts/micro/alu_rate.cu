// Microbenchmark: per-SMSP issue rate of the softmax instruction mix (MUFU.EX2, FFMA2, FADD2,
// F2FP bf16 pack, scalar FFMA, FMNMX3).  One CTA of W warps; each thread runs 8 independent chains.
// Prints cycles per warp-instruction per SMSP (W/4 warps share one SMSP).
#include "../../paper_2603_18636_b200/csrc/common.cuh"
#include <cstdio>
using namespace cs;

template <int MODE>
__global__ void k(float* out, long long* cyc, int iters) {
  float2 a[8];
  uint32_t u[8];
  for (int i = 0; i < 8; ++i) { a[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f); u[i] = i; }
  const float2 c2 = make_float2(0.999f, 0.999f), d2 = make_float2(1e-3f, 1e-3f);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) { a[i].x = ex2(a[i].x); }
      if (MODE == 1) { a[i] = ffma2(a[i], c2, d2); }
      if (MODE == 2) { a[i] = fadd2(a[i], d2); }
      if (MODE == 3) { u[i] ^= pack_bf16x2(a[i].x, a[i].y); }
      if (MODE == 4) { a[i].x = fmaf(a[i].x, 0.999f, 1e-3f); }
      if (MODE == 5) { a[i].x = fmax3(a[i].x, a[i].y, d2.x); }
      if (MODE == 6) { a[i] = ex2_poly2(a[i]); }
      if (MODE == 7) { asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(u[i])); }
      if (MODE == 8) { asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(u[i])); }
      if (MODE == 9) { asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(u[i]) : "f"(a[i].x), "f"(__uint_as_float(u[i]))); }
      if (MODE == 10) {  // softmax pair via bf16x2 ex2: ffma2, pack, ex2, unpack, fadd2
        const float2 x = ffma2(a[i], c2, d2);
        uint32_t h;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(x.y), "f"(x.x));
        asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h));
        u[i] ^= h;
        a[i] = fadd2(a[i], make_float2(__uint_as_float(h << 16), __uint_as_float(h & 0xffff0000u)));
      }
      if (MODE == 12) {  // the attention's pair mix: 3 of 4 pairs on MUFU, 1 on the polynomial
        const float2 x = ffma2(a[i], c2, d2);
        const float2 p = (i & 3) == 3 ? ex2_poly2(x) : make_float2(ex2(x.x), ex2(x.y));
        a[i] = fadd2(a[i], p);
        u[i] ^= pack_bf16x2(p.x, p.y);
      }
      if (MODE == 11) {  // current pair: ffma2, 2x ex2 f32, fadd2, pack
        const float2 x = ffma2(a[i], c2, d2);
        const float2 p = make_float2(ex2(x.x), ex2(x.y));
        a[i] = fadd2(a[i], p);
        u[i] ^= pack_bf16x2(p.x, p.y);
      }
    }
  }
  long long t1 = clock64();
  float s = 0.f;
  for (int i = 0; i < 8; ++i) s += a[i].x + a[i].y + (float)u[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// One row's worth of softmax pairs per iteration: NP independent pairs (x from a register array),
// the kernel's mix (3 of 4 pairs on MUFU, 1 on the polynomial), 4 FADD2 sum chains, bf16 pack.
template <int NP>
__global__ void k_wide(float* out, long long* cyc, int iters) {
  float2 s[NP];
  for (int i = 0; i < NP; ++i) s[i] = make_float2(-(threadIdx.x & 7) * 0.1f - i * 0.01f, -i * 0.02f);
  float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
  uint32_t pk = 0;
  const float2 sl2 = make_float2(0.1275f, 0.1275f);
  float m = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const float2 nm2 = make_float2(-m, -m);
#pragma unroll
    for (int c = 0; c < NP; ++c) {
      const float2 x = ffma2(s[c], sl2, nm2);
      const float2 p = (c & 3) == 3 ? ex2_poly2(x) : make_float2(ex2(x.x), ex2(x.y));
      acc[c & 3] = fadd2(acc[c & 3], p);
      pk ^= pack_bf16x2(p.x, p.y);
    }
    m += 1e-7f * acc[0].x;  // next iteration depends on this one (like the next tile on the max)
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc[0].x + acc[1].y + acc[2].x + acc[3].y + (float)pk;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int NP>
void run_wide(int warps) {
  float* out; long long* cyc;
  cudaMalloc(&out, 1024 * 4 * 148); cudaMalloc(&cyc, 8 * 148);
  const int iters = 1024;
  k_wide<NP><<<148, warps * 32>>>(out, cyc, 16);
  k_wide<NP><<<148, warps * 32>>>(out, cyc, iters);
  long long c = 0;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("wide NP=%2d warps=%2d  cycles per pair per SMSP: %.2f  (per row of %d pairs per warp: %.0f)\n", NP, warps,
         (double)c / (iters * (double)NP) / (warps / 4.0), NP, (double)c / iters);
  cudaFree(out); cudaFree(cyc);
}

template <int MODE>
void run(const char* name, int warps) {
  float* out; long long* cyc;
  cudaMalloc(&out, 1024 * 4 * 148); cudaMalloc(&cyc, 8 * 148);
  const int iters = 4096;
  k<MODE><<<148, warps * 32>>>(out, cyc, 16);
  k<MODE><<<148, warps * 32>>>(out, cyc, iters);
  long long c = 0;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  // instructions per warp = iters * 8 (poly: per pair of values)
  const double per = (double)c / (iters * 8.0) / (warps / 4.0);
  printf("%-10s warps=%2d  cycles per warp-instr per SMSP: %.2f\n", name, warps, per);
  cudaFree(out); cudaFree(cyc);
}

int main(int argc, char** argv) {
  if (argc > 1) {
    for (int w : {4, 8, 16}) { run_wide<16>(w); run_wide<32>(w); run_wide<64>(w); }
    return 0;
  }
  for (int w : {4, 8, 16, 32}) {
    run<0>("mufu.ex2", w); run<1>("ffma2", w); run<2>("fadd2", w); run<3>("f2fp", w);
    run<4>("ffma", w); run<5>("fmnmx3", w); run<6>("poly2", w);
    run<7>("ex2.bf16x2", w); run<8>("ex2.f16x2", w); run<9>("cvt.bf16x2", w);
    run<10>("pair.bf16", w); run<11>("pair.f32", w); run<12>("pair.mix", w);
  }
  return 0;
}
