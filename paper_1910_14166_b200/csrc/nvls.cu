// a3 over NVLink SHARP: the [SA | g] exchange as ONE kernel on
// a multicast (NVLS) mapping of a symmetric buffer -- every rank's copy of the
// buffer is bound to one multicast address, so `multimem.ld_reduce.add.f64`
// returns the sum of all ranks' copies of an element (the switch reduces) and
// `multimem.st` writes a value to every rank's copy.  Rank r reduces and
// broadcasts slice r of the buffer; the ranks meet at a barrier before (their
// partial sketches are written) and after (every slice's broadcast has
// landed).  The sum is exact by linearity of S (the per-rank
// S_k A_k with global-row hashes sum to S A); its rounding is the switch's
// order, the same on every rank (one value is broadcast to all).
//
// The symmetric buffer, its multicast mapping and the per-rank signal pads
// come from the caller (torch symmetric memory: plumbing); this file holds
// only the exchange's arithmetic and its barrier.
#include "common.cuh"
#include "kernels.h"

namespace ihs {

namespace {
constexpr int kNvlsThreads = 512;

// Signal slots: pad[b * world + r] on rank p is set by rank r for block b (a
// compare-and-swap 0 -> 1 that waits until the slot is free) and cleared by
// rank p when it waits (1 -> 0), so the same slots serve every barrier.
__device__ __forceinline__ void put_signal(uint32_t *slot) {
  while (atomicCAS_system(slot, 0u, 1u) != 0u) {
  }
}
__device__ __forceinline__ void wait_signal(uint32_t *slot) {
  while (atomicCAS_system(slot, 1u, 0u) != 1u) {
  }
}

// All ranks' block `blk` meet: thread p < world signals rank p and waits for
// rank p's signal.  Release before (this rank's writes are visible system
// wide), acquire after.
__device__ __forceinline__ void block_barrier(uint32_t *const *pads, int rank, int world, int blk) {
  __syncthreads();
  if ((int)threadIdx.x < world) {
    __threadfence_system();
    put_signal(pads[threadIdx.x] + (size_t)blk * world + rank);
    wait_signal(pads[rank] + (size_t)blk * world + threadIdx.x);
    __threadfence_system();
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kNvlsThreads) nvls_allreduce_kernel(double *mc, uint32_t *const *pads, int rank,
                                                                     int world, int64_t count) {
  block_barrier(pads, rank, world, blockIdx.x);
  const int64_t lo = count * rank / world, hi = count * (rank + 1) / world;
  for (int64_t i = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < hi; i += (int64_t)gridDim.x * blockDim.x) {
    double v;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f64 %0, [%1];" : "=d"(v) : "l"(mc + i) : "memory");
    asm volatile("multimem.st.relaxed.sys.global.f64 [%0], %1;" ::"l"(mc + i), "d"(v) : "memory");
  }
  block_barrier(pads, rank, world, blockIdx.x);
}
}  // namespace

int nvls_blocks(int64_t count, int world, int num_sms) {
  const int64_t per_rank = (count + world - 1) / std::max(world, 1);
  return (int)std::max<int64_t>(1, std::min<int64_t>((per_rank + kNvlsThreads - 1) / kNvlsThreads, num_sms));
}

cudaError_t launch_nvls_allreduce(double *mc, uint32_t *const *pads, int rank, int world, int64_t count, int blocks,
                                  cudaStream_t st, LaunchCounter lc) {
  nvls_allreduce_kernel<<<blocks, kNvlsThreads, 0, st>>>(mc, pads, rank, world, count);
  lc.add();
  return cudaGetLastError();
}

}  // namespace ihs
