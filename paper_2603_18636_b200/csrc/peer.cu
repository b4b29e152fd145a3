// peer.cu — cross-process peer memory for the fused Ulysses return path:
//   CUDA IPC handle export / import of caller-owned device buffers (any pointer inside an
//   allocation: the handle names the allocation, the offset is carried separately), and a
//   device-side barrier over per-rank flag arrays in peer memory, so the consumer of a token
//   block written by the other ranks' attention epilogues waits on the GPU, not on the host.
#include "kernels.cuh"

namespace cs {

// One warp: lane p < P stores `epoch` into flags_p[rank] (system-scope release), then spins on
// its own flags[p] until rank p has signalled the same epoch.  A wait beyond ~2^32 cycles traps
// (a dead peer fails the launch instead of hanging the GPU).
__global__ void k_peer_barrier(int P, int rank, const uint64_t* __restrict__ peer_flags, int epoch) {
  const int p = threadIdx.x;
  __threadfence_system();  // this stream's earlier peer stores are visible before the signal
  __syncwarp();
  if (p < P) {
    int* remote = reinterpret_cast<int*>(peer_flags[p]) + rank;
    asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(remote), "r"(epoch) : "memory");
    const int* mine = reinterpret_cast<const int*>(peer_flags[rank]) + p;
    const long long t0 = clock64();
    int v = 0;
    do {
      asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(mine) : "memory");
      if (clock64() - t0 > (1LL << 32)) __trap();
    } while (v < epoch);
  }
  __syncwarp();
}

cudaError_t launch_peer_barrier(int P, int rank, const uint64_t* peer_flags, int epoch, cudaStream_t st) {
  k_peer_barrier<<<1, 32, 0, st>>>(P, rank, peer_flags, epoch);
  return cudaGetLastError();
}

}  // namespace cs
