// a2 (+ a5 fused) for dense CountSketch, TMA-fed: one CTA per bucket.  Thread 0
// streams the bucket's rows (ascending, from the stable sort) into a 3-stage
// shared-memory ring with 1-D bulk copies (cp.async.bulk -> UBLKCP), one per
// row, completing on an mbarrier per stage.  Each thread owns one column: it
// adds sign*A[row, c] for the rows of a stage in ring order, i.e. the same
// left-to-right fp64 sum as the oracle (SA bit-identical at P = 1).  With the
// gradient fused, each warp first reduces the dot products a_i.x of its rows
// of the stage (r_i = b_i - a_i.x to shared memory), then every thread also
// accumulates g_c += r_i A[i, c].  A is read from HBM once per iteration.
//
// PAPER.md:236-240 (stream A; bucket h(i) accumulates +-row i) and Eq. (2),
// PAPER.md:83-86 (the linear term A^T(b - A x^t)).
#include "common.cuh"
#include "kernels.h"

namespace ihs {

namespace {
constexpr int kScanTile = 4096;
constexpr int kStages = 3;
constexpr int kRows = 8;  // rows per stage

__device__ __forceinline__ int32_t scanned_at(const int32_t *hist, const int32_t *tile_sums, int64_t e) {
  return hist[e] + tile_sums[e / kScanTile];
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Warps 0-3 consume (one column per thread, two for d > 128); warp 4 produces:
// it prefetches the perm entries of the next stage, waits until the stage's
// slot is released (empty barrier, one arrival per consumer warp) and issues
// one bulk copy per row, completing on the slot's full barrier.
constexpr int kConsumers = 128;
template <bool FUSE>
__global__ void __launch_bounds__(kConsumers + 32, 7) cs_gather_tma_kernel(
    const double *__restrict__ A, int64_t n, int d, int m, const int32_t *__restrict__ hist,
    const int32_t *__restrict__ tile_sums, int64_t nchunks, const uint32_t *__restrict__ perm,
    const double *__restrict__ bvec, const double *__restrict__ x, double *__restrict__ SA,
    double *__restrict__ gpart) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double *ring = reinterpret_cast<double *>(smem_raw);                                // [kStages][kRows][d]
  uint64_t *full = reinterpret_cast<uint64_t *>(ring + (size_t)kStages * kRows * d);  // [kStages]
  uint64_t *empty = full + kStages;                                                   // [kStages]
  uint32_t *rid = reinterpret_cast<uint32_t *>(empty + kStages);                      // [kStages][kRows]
  double *res = reinterpret_cast<double *>(rid + kStages * kRows);                    // [kStages][kRows]
  const int b = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t beg = scanned_at(hist, tile_sums, (int64_t)b * nchunks);
  const int64_t end = (b + 1 < m) ? scanned_at(hist, tile_sums, (int64_t)(b + 1) * nchunks) : n;
  const int64_t len = end - beg;
  const int64_t nb = (len + kRows - 1) / kRows;
  const uint32_t row_bytes = (uint32_t)d * 8u;

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumers / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kConsumers / 32) {
    // ---------------- producer warp
    auto perm_of = [&](int64_t k) -> uint32_t {
      const int64_t i = k * kRows + lane;
      return (lane < kRows && k < nb && i < len) ? perm[beg + i] : 0u;
    };
    uint32_t e = perm_of(0);
    for (int64_t k = 0; k < nb; ++k) {
      const int s = (int)(k % kStages);
      const int cnt = (int)min((int64_t)kRows, len - k * kRows);
      const uint32_t enext = perm_of(k + 1);  // in flight while we wait for the slot
      if (k >= kStages) mbar_wait(&empty[s], (uint32_t)(((k / kStages) - 1) & 1));
      if (lane < cnt) rid[s * kRows + lane] = e;
      __syncwarp();
      if (lane == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&full[s], (uint32_t)cnt * row_bytes);
      }
      __syncwarp();
      if (lane < cnt)
        bulk_g2s(ring + ((size_t)s * kRows + lane) * d, A + (int64_t)(e & 0x7fffffffu) * d, row_bytes, &full[s]);
      e = enext;
    }
    return;
  }
  // ---------------- consumer warps
  const int c0 = tid, c1 = tid + kConsumers;
  const bool v0 = c0 < d, v1 = c1 < d;
  double acc0 = 0.0, acc1 = 0.0, g0 = 0.0, g1 = 0.0;
  double xv[8];
  if constexpr (FUSE) {
#pragma unroll
    for (int q = 0; q < 8; ++q) xv[q] = (lane + 32 * q < d) ? x[lane + 32 * q] : 0.0;
  }
  for (int64_t k = 0; k < nb; ++k) {
    const int s = (int)(k % kStages);
    const int cnt = (int)min((int64_t)kRows, len - k * kRows);
    mbar_wait(&full[s], (uint32_t)((k / kStages) & 1));
    const double *st = ring + (size_t)s * kRows * d;
    if constexpr (FUSE) {
      for (int r = warp; r < cnt; r += kConsumers / 32) {
        const double *row = st + (size_t)r * d;
        double p = 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (lane + 32 * q < d) p = fma(row[lane + 32 * q], xv[q], p);
        p = warp_sum(p);
        if (lane == 0) res[s * kRows + r] = bvec[rid[s * kRows + r] & 0x7fffffffu] - p;
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory");
    }
#pragma unroll 4
    for (int r = 0; r < cnt; ++r) {
      const double *row = st + (size_t)r * d;
      const bool neg = (rid[s * kRows + r] >> 31) != 0;
      if (v0) {
        const double a = row[c0];
        acc0 += neg ? -a : a;
        if constexpr (FUSE) g0 = fma(res[s * kRows + r], a, g0);
      }
      if (v1) {
        const double a = row[c1];
        acc1 += neg ? -a : a;
        if constexpr (FUSE) g1 = fma(res[s * kRows + r], a, g1);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  if (v0) {
    SA[(int64_t)b * d + c0] = acc0;
    if constexpr (FUSE) gpart[(int64_t)b * d + c0] = g0;
  }
  if (v1) {
    SA[(int64_t)b * d + c1] = acc1;
    if constexpr (FUSE) gpart[(int64_t)b * d + c1] = g1;
  }
}
}  // namespace

bool cs_gather_tma_supported(int64_t d, const void *A) {
  return d >= 2 && d <= 256 && (d % 2) == 0 && (reinterpret_cast<uintptr_t>(A) % 16) == 0;
}

cudaError_t launch_cs_gather_tma(const double *A, int64_t n, int64_t d, int64_t m, const int32_t *hist,
                                 const int32_t *tile_sums, int64_t nchunks, const uint32_t *perm, const double *bvec,
                                 const double *x, double *SA, double *gpart, cudaStream_t st, LaunchCounter lc) {
  const size_t smem = (size_t)kStages * kRows * d * 8 + 2 * kStages * 8 + kStages * kRows * 4 + kStages * kRows * 8 + 64;
  if (gpart) {
    IHS_SMEM_ATTR(cs_gather_tma_kernel<true>, smem);
    cs_gather_tma_kernel<true><<<(unsigned)m, kConsumers + 32, smem, st>>>(A, n, (int)d, (int)m, hist, tile_sums, nchunks,
                                                                    perm, bvec, x, SA, gpart);
  } else {
    IHS_SMEM_ATTR(cs_gather_tma_kernel<false>, smem);
    cs_gather_tma_kernel<false><<<(unsigned)m, kConsumers + 32, smem, st>>>(A, n, (int)d, (int)m, hist, tile_sums, nchunks,
                                                                     perm, nullptr, nullptr, SA, nullptr);
  }
  lc.add();
  return cudaGetLastError();
}

}  // namespace ihs
