// a2 (+ a5 fused, NEXT-1 single pass) for dense CountSketch: one warp per
// (bucket, 32*NV-column slice) walks the bucket's rows in ascending row order
// (the stable sort of cs_sort.cu) and sums sign*row in registers -- the same
// left-to-right fp64 sum as the oracle's loop, so SA is bit-identical to it at
// P = 1.  With the gradient fused, the same loaded rows also give
// r_i = b_i - a_i.x (transpose-reduced across the warp) and g += r_i a_i, so A
// is read from HBM once per IHS iteration.
//
// PAPER.md:236-240 (section 2: stream A, bucket h(i) accumulates +-row i) and
// Eq. (2), PAPER.md:83-86 (the linear term A^T(b - A x^t)).
#include "common.cuh"
#include "kernels.h"

#include <cstdlib>

namespace ihs {

namespace {
constexpr int kScanTile = 4096;

__device__ __forceinline__ int32_t scanned_at(const int32_t *hist, const int32_t *tile_sums, int64_t e) {
  return hist[e] + tile_sums[e / kScanTile];
}

// Rows of a bucket are consumed in batches of U.  Batch k+1's rows are loaded
// while batch k is reduced (two register buffers), and the perm entries are
// fetched two batches ahead, so each warp keeps 2*U rows in flight.  Loads are
// never predicated: a predicated load followed by a zero-fill of the same
// register serialises on the scoreboard.  Out-of-range columns read column
// d-1 (and carry x = 0); out-of-range rows re-read the bucket's last row and
// are skipped by the accumulations.
template <int NV, int U, bool FUSE>
struct GatherWarp {
  const double *__restrict__ A;
  const uint32_t *__restrict__ perm;
  const double *__restrict__ bvec;
  int64_t beg, len;
  int d, lane;
  int colc[NV];
  double acc[NV], gacc[NV], xv[NV];

  // L2 streaming: the rows of bucket b ascend, and all warps move through A at
  // about the same rate, so the union of their reads is a band moving down A.
  // Each warp owns a 1/nwarps sub-chunk of every window of `win_rows` rows and,
  // when it first enters window w, prefetches its sub-chunk of window w + pd
  // with one bulk L2 prefetch (UBLKPF): A then streams from HBM in large
  // sequential pieces and the bucket-ordered row reads hit L2.
  int64_t n, win_rows, pd, last_win, chunk;
  int wid;
  __device__ __forceinline__ void prefetch_window(int64_t v) const {
    const int64_t r0 = v * win_rows + (int64_t)wid * chunk;
    const int64_t r1 = min(min(r0 + chunk, (v + 1) * win_rows), n);
    if (r0 < r1)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(A + r0 * d), "r"((uint32_t)((r1 - r0) * d * 8))
                   : "memory");
  }
  __device__ __forceinline__ void advance(uint32_t pk) {
    if (win_rows <= 0) return;
    const int64_t row = (int64_t)(__shfl_sync(0xffffffffu, pk, 0) & 0x7fffffffu);
    const int64_t w = row / win_rows;
    if (w > last_win) {
      if (lane == 0)
        for (int64_t v = max(last_win + 1, w - 1) + pd; v <= w + pd; ++v) prefetch_window(v);
      last_win = w;
    }
  }
  __device__ __forceinline__ uint32_t perm_at(int64_t k) const {
    int64_t i = k * U + (lane & (U - 1));
    return perm[beg + (i < len ? i : len - 1)];
  }
  __device__ __forceinline__ void load(double (&v)[U][NV], uint32_t pk) const {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t e = __shfl_sync(0xffffffffu, pk, u);
      const double *rowp = A + (int64_t)(e & 0x7fffffffu) * d;
#pragma unroll
      for (int k = 0; k < NV; ++k) v[u][k] = ldg_stream(rowp + colc[k]);
    }
  }
  __device__ __forceinline__ void process(const double (&v)[U][NV], uint32_t pk, int64_t k) {
    const int cnt = (int)min((int64_t)U, len - k * U);
    if constexpr (FUSE) {
      double p[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        p[u] = 0.0;
#pragma unroll
        for (int c = 0; c < NV; ++c) p[u] = fma(v[u][c], xv[c], p[u]);
      }
      transpose_reduce<U>(p, lane);
      const int myu = reduced_row_of_lane<U>(lane);
      const uint32_t me = __shfl_sync(0xffffffffu, pk, myu);
      const double res = (myu < cnt) ? bvec[me & 0x7fffffffu] - p[0] : 0.0;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const double ru = __shfl_sync(0xffffffffu, res, owner_lane_of_row<U>(u));
#pragma unroll
        for (int c = 0; c < NV; ++c) gacc[c] = fma(ru, v[u][c], gacc[c]);
      }
    }
    // ascending rows of the bucket: the oracle's summation order
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t e = __shfl_sync(0xffffffffu, pk, u);
      if (u < cnt) {
        const bool neg = (e >> 31) != 0;
#pragma unroll
        for (int c = 0; c < NV; ++c) acc[c] += neg ? -v[u][c] : v[u][c];
      }
    }
  }
};

template <int NV, int U, bool FUSE>
__global__ void __launch_bounds__(64) cs_gather_kernel(const double *__restrict__ A, int64_t n, int d, int m,
                                                       int nslices, const int32_t *__restrict__ hist,
                                                       const int32_t *__restrict__ tile_sums, int64_t nchunks,
                                                       const uint32_t *__restrict__ perm,
                                                       const double *__restrict__ bvec,
                                                       const double *__restrict__ x, double *__restrict__ SA,
                                                       double *__restrict__ gpart, int64_t win_rows, int64_t pd,
                                                       double scale) {
  const int warp = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (warp >= m * nslices) return;
  const int b = warp / nslices;
  const int slice = warp - b * nslices;
  const int64_t beg = scanned_at(hist, tile_sums, (int64_t)b * nchunks);
  const int64_t end = (b + 1 < m) ? scanned_at(hist, tile_sums, (int64_t)(b + 1) * nchunks) : n;

  GatherWarp<NV, U, FUSE> w;
  w.A = A;
  w.perm = perm;
  w.bvec = bvec;
  w.beg = beg;
  w.len = end - beg;
  w.d = d;
  w.lane = lane;
  int col[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    col[k] = slice * 32 * NV + lane + 32 * k;
    w.colc[k] = col[k] < d ? col[k] : d - 1;
    w.acc[k] = 0.0;
    w.gacc[k] = 0.0;
    w.xv[k] = (FUSE && col[k] < d) ? x[col[k]] : 0.0;
  }
  w.n = n;
  w.win_rows = win_rows;
  w.pd = pd;
  w.wid = warp;
  w.chunk = win_rows > 0 ? (win_rows + (int64_t)m * nslices - 1) / ((int64_t)m * nslices) : 0;
  w.last_win = -1;
  const int64_t nb = (w.len + U - 1) / U;
  if (nb > 0) {
    double va[U][NV], vb[U][NV];
    uint32_t p0 = w.perm_at(0), p1 = w.perm_at(1 < nb ? 1 : 0);
    if (win_rows > 0) {  // initial fill: windows w0 + 1 .. w0 + pd
      const int64_t w0 = (int64_t)(__shfl_sync(0xffffffffu, p0, 0) & 0x7fffffffu) / win_rows;
      if (lane == 0)
        for (int64_t v = w0 + 1; v <= w0 + pd; ++v) w.prefetch_window(v);
      w.last_win = w0;
    }
    w.load(va, p0);
#pragma unroll 1
    for (int64_t k = 0; k < nb; k += 2) {
      const uint32_t p2 = w.perm_at(k + 2 < nb ? k + 2 : nb - 1);
      if (k + 1 < nb) {
        w.advance(p1);
        w.load(vb, p1);
      }
      w.process(va, p0, k);
      const uint32_t p3 = w.perm_at(k + 3 < nb ? k + 3 : nb - 1);
      if (k + 2 < nb) {
        w.advance(p2);
        w.load(va, p2);
      }
      if (k + 1 < nb) w.process(vb, p1, k + 1);
      p0 = p2;
      p1 = p3;
    }
  }
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    if (col[k] < d) {
      SA[(int64_t)b * d + col[k]] = scale == 1.0 ? w.acc[k] : w.acc[k] * scale;
      if constexpr (FUSE) gpart[(int64_t)b * d + col[k]] = w.gacc[k];
    }
  }
}

// cp.async-fed variant (LDGSTS, 16-byte pieces, L1 bypass): each warp keeps a
// private ring of S stages x U rows in shared memory, so S-1 batches (16 KiB at
// d = 128) stay in flight without holding registers; the register-staged
// kernel above is capped by the register file at ~7 warps per SM.  Rows are
// consumed from the ring in ascending order exactly as above (bit-exact SA).
// Requires even d and a 16-byte aligned A.
template <int NV, int U, int S, bool FUSE>
__global__ void __launch_bounds__(64) cs_gather_async_kernel(const double *__restrict__ A, int64_t n, int d, int m,
                                                             const int32_t *__restrict__ hist,
                                                             const int32_t *__restrict__ tile_sums, int64_t nchunks,
                                                             const uint32_t *__restrict__ perm,
                                                             const double *__restrict__ bvec,
                                                             const double *__restrict__ x, double *__restrict__ SA,
                                                             double *__restrict__ gpart, double scale) {
  extern __shared__ __align__(16) double ring_all[];
  const int wib = threadIdx.x >> 5;
  const int b = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (b >= m) return;
  double *ring = ring_all + (size_t)wib * S * U * d;
  const int64_t beg = scanned_at(hist, tile_sums, (int64_t)b * nchunks);
  const int64_t end = (b + 1 < m) ? scanned_at(hist, tile_sums, (int64_t)(b + 1) * nchunks) : n;
  const int64_t len = end - beg;
  const int64_t nb = (len + U - 1) / U;
  const int pieces = d / 2;  // 16-byte pieces per row
  int col[NV], colc[NV];
  double acc[NV], gacc[NV], xv[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    col[k] = lane + 32 * k;
    colc[k] = col[k] < d ? col[k] : d - 1;
    acc[k] = 0.0;
    gacc[k] = 0.0;
    xv[k] = (FUSE && col[k] < d) ? x[col[k]] : 0.0;
  }
  auto perm_at = [&](int64_t k) -> uint32_t {
    const int64_t i = k * U + (lane & (U - 1));
    return perm[beg + (i < len ? i : (len > 0 ? len - 1 : 0))];
  };
  auto issue = [&](int64_t k, uint32_t pk) {
    if (k < nb) {
      double *dst = ring + (size_t)(k % S) * U * d;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t e = __shfl_sync(0xffffffffu, pk, u);
        const char *src = reinterpret_cast<const char *>(A + (int64_t)(e & 0x7fffffffu) * d);
        char *dr = reinterpret_cast<char *>(dst + (size_t)u * d);
        for (int p = lane; p < pieces; p += 32) {
          const unsigned sa = (unsigned)__cvta_generic_to_shared(dr + 16 * p);
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(src + 16 * p) : "memory");
        }
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  if (nb > 0) {
    // prologue: batches 0 .. S-2 in flight; perm entries are fetched one batch ahead
    uint32_t pcur = perm_at(0);
#pragma unroll
    for (int k = 0; k < S - 1; ++k) {
      const uint32_t pn = perm_at(k + 1 < nb ? k + 1 : nb - 1);
      issue(k, pcur);
      pcur = pn;
    }
    uint32_t pissue = pcur;  // perm entries of batch S-1
#pragma unroll 1
    for (int64_t k = 0; k < nb; ++k) {
      const uint32_t pnext = perm_at(k + S < nb ? k + S : nb - 1);
      issue(k + S - 1, pissue);
      pissue = pnext;
      asm volatile("cp.async.wait_group %0;" ::"n"(S - 1) : "memory");
      __syncwarp();
      const double *st = ring + (size_t)(k % S) * U * d;
      const uint32_t pk = perm_at(k);
      const int cnt = (int)min((int64_t)U, len - k * U);
      double v[U][NV];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int c = 0; c < NV; ++c) v[u][c] = st[(size_t)(u < cnt ? u : 0) * d + colc[c]];
      if constexpr (FUSE) {
        double p[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          p[u] = 0.0;
#pragma unroll
          for (int c = 0; c < NV; ++c) p[u] = fma(v[u][c], xv[c], p[u]);
        }
        transpose_reduce<U>(p, lane);
        const int myu = reduced_row_of_lane<U>(lane);
        const uint32_t me = __shfl_sync(0xffffffffu, pk, myu);
        const double res = (myu < cnt) ? bvec[me & 0x7fffffffu] - p[0] : 0.0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const double ru = __shfl_sync(0xffffffffu, res, owner_lane_of_row<U>(u));
#pragma unroll
          for (int c = 0; c < NV; ++c) gacc[c] = fma(ru, v[u][c], gacc[c]);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t e = __shfl_sync(0xffffffffu, pk, u);
        if (u < cnt) {
          const bool neg = (e >> 31) != 0;
#pragma unroll
          for (int c = 0; c < NV; ++c) acc[c] += neg ? -v[u][c] : v[u][c];
        }
      }
      __syncwarp();  // the slot is refilled by the next iteration's issue
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
  }
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    if (col[k] < d) {
      SA[(int64_t)b * d + col[k]] = scale == 1.0 ? acc[k] : acc[k] * scale;
      if constexpr (FUSE) gpart[(int64_t)b * d + col[k]] = gacc[k];
    }
  }
}

template <int NV, int U, int S>
cudaError_t launch_async_t(bool fuse, const double *A, int64_t n, int d, int m, const int32_t *hist,
                           const int32_t *tile_sums, int64_t nchunks, const uint32_t *perm, const double *bvec,
                           const double *x, double *SA, double *gpart, double scale, cudaStream_t st) {
  const size_t smem = (size_t)2 * S * U * d * 8;
  const unsigned grid = (unsigned)((m + 1) / 2);
  if (fuse) {
    IHS_SMEM_ATTR((cs_gather_async_kernel<NV, U, S, true>), smem);
    cs_gather_async_kernel<NV, U, S, true><<<grid, 64, smem, st>>>(A, n, d, m, hist, tile_sums, nchunks, perm, bvec,
                                                                   x, SA, gpart, scale);
  } else {
    IHS_SMEM_ATTR((cs_gather_async_kernel<NV, U, S, false>), smem);
    cs_gather_async_kernel<NV, U, S, false><<<grid, 64, smem, st>>>(A, n, d, m, hist, tile_sums, nchunks, perm,
                                                                    nullptr, nullptr, SA, nullptr, scale);
  }
  return cudaGetLastError();
}

template <int NV, int U>
cudaError_t launch_nv(bool fuse, const double *A, int64_t n, int d, int m, int nslices, const int32_t *hist,
                      const int32_t *tile_sums, int64_t nchunks, const uint32_t *perm, const double *bvec,
                      const double *x, double *SA, double *gpart, double scale, cudaStream_t st) {
  const int64_t warps = (int64_t)m * nslices;
  // L2 streaming window (IHS_L2_WIN_MB / IHS_L2_PD): off by default -- measured slower on B200
  static const int64_t win_mb = getenv("IHS_L2_WIN_MB") ? atoll(getenv("IHS_L2_WIN_MB")) : 0;
  static const int64_t pd = getenv("IHS_L2_PD") ? atoll(getenv("IHS_L2_PD")) : 2;
  const int64_t win_rows = win_mb > 0 ? std::max<int64_t>(1, (win_mb << 20) / (8 * (int64_t)d)) : 0;
  const unsigned grid = (unsigned)((warps + 1) / 2);
  if (fuse)
    cs_gather_kernel<NV, U, true><<<grid, 64, 0, st>>>(A, n, d, m, nslices, hist, tile_sums, nchunks, perm, bvec, x,
                                                        SA, gpart, win_rows, pd, scale);
  else
    cs_gather_kernel<NV, U, false><<<grid, 64, 0, st>>>(A, n, d, m, nslices, hist, tile_sums, nchunks, perm,
                                                         nullptr, nullptr, SA, nullptr, win_rows, pd, scale);
  return cudaGetLastError();
}
}  // namespace

bool cs_gather_async_supported(int64_t d, const void *A) {
  return d >= 2 && d <= 256 && (d % 2) == 0 && (reinterpret_cast<uintptr_t>(A) % 16) == 0;
}

cudaError_t launch_cs_gather_async(const double *A, int64_t n, int64_t d, int64_t m, const int32_t *hist,
                                   const int32_t *tile_sums, int64_t nchunks, const uint32_t *perm,
                                   const double *bvec, const double *x, double *SA, double *gpart, double scale,
                                   cudaStream_t st, LaunchCounter lc) {
  const bool fuse = gpart != nullptr;
  const int nv = (int)((d + 31) / 32);
  static const int stages = getenv("IHS_ASYNC_STAGES") ? atoi(getenv("IHS_ASYNC_STAGES")) : 3;
  cudaError_t e;
  const int di = (int)d, mi = (int)m;
#define IHS_ASYNC(NV, U)                                                                                          \
  (stages >= 4                                                                                                   \
       ? launch_async_t<NV, U, 4>(fuse, A, n, di, mi, hist, tile_sums, nchunks, perm, bvec, x, SA, gpart, scale, st) \
       : launch_async_t<NV, U, 3>(fuse, A, n, di, mi, hist, tile_sums, nchunks, perm, bvec, x, SA, gpart, scale, st))
  switch (nv) {
    case 1: e = IHS_ASYNC(1, 8); break;
    case 2: e = IHS_ASYNC(2, 8); break;
    case 3: e = IHS_ASYNC(3, 8); break;
    case 4: e = IHS_ASYNC(4, 8); break;
    case 5:
    case 6: e = IHS_ASYNC(6, 4); break;
    default: e = IHS_ASYNC(8, 4); break;
  }
#undef IHS_ASYNC
  lc.add();
  return e;
}

cudaError_t launch_cs_gather(const double *A, int64_t n, int64_t d, int64_t m, const int32_t *hist,
                             const int32_t *tile_sums, int64_t nchunks, const uint32_t *perm, const double *bvec,
                             const double *x, double *SA, double *gpart, double scale, cudaStream_t st,
                             LaunchCounter lc) {
  const bool fuse = gpart != nullptr;
  int nv = (int)((d + 31) / 32);
  int nslices = 1;
  if (nv > 8) {
    if (fuse) return cudaErrorInvalidValue;  // fused path needs a whole row per warp
    nslices = (int)((d + 255) / 256);
    nv = 8;
  }
  cudaError_t e;
  const int di = (int)d, mi = (int)m;
  switch (nv) {
    case 1: e = launch_nv<1, 16>(fuse, A, n, di, mi, nslices, hist, tile_sums, nchunks, perm, bvec, x, SA, gpart, scale, st); break;
    case 2: e = launch_nv<2, 16>(fuse, A, n, di, mi, nslices, hist, tile_sums, nchunks, perm, bvec, x, SA, gpart, scale, st); break;
    case 3: e = launch_nv<3, 8>(fuse, A, n, di, mi, nslices, hist, tile_sums, nchunks, perm, bvec, x, SA, gpart, scale, st); break;
    case 4: e = launch_nv<4, 8>(fuse, A, n, di, mi, nslices, hist, tile_sums, nchunks, perm, bvec, x, SA, gpart, scale, st); break;
    case 5:
    case 6: e = launch_nv<6, 4>(fuse, A, n, di, mi, nslices, hist, tile_sums, nchunks, perm, bvec, x, SA, gpart, scale, st); break;
    default: e = launch_nv<8, 4>(fuse, A, n, di, mi, nslices, hist, tile_sums, nchunks, perm, bvec, x, SA, gpart, scale, st); break;
  }
  lc.add();
  return e;
}

}  // namespace ihs
