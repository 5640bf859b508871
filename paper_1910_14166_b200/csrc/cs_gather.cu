// a2 (+ a5 fused, NEXT-1 single pass) for dense CountSketch where the TMA
// gather (cs_gather_tma.cu) does not apply (odd d, d > 256, an A not 16-byte
// aligned): one warp per
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
                                                       double *__restrict__ gpart, double scale) {
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
  const int64_t nb = (w.len + U - 1) / U;
  if (nb > 0) {
    double va[U][NV], vb[U][NV];
    uint32_t p0 = w.perm_at(0), p1 = w.perm_at(1 < nb ? 1 : 0);
    w.load(va, p0);
#pragma unroll 1
    for (int64_t k = 0; k < nb; k += 2) {
      const uint32_t p2 = w.perm_at(k + 2 < nb ? k + 2 : nb - 1);
      if (k + 1 < nb) w.load(vb, p1);
      w.process(va, p0, k);
      const uint32_t p3 = w.perm_at(k + 3 < nb ? k + 3 : nb - 1);
      if (k + 2 < nb) w.load(va, p2);
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

template <int NV, int U>
cudaError_t launch_nv(bool fuse, const double *A, int64_t n, int d, int m, int nslices, const int32_t *hist,
                      const int32_t *tile_sums, int64_t nchunks, const uint32_t *perm, const double *bvec,
                      const double *x, double *SA, double *gpart, double scale, cudaStream_t st) {
  const int64_t warps = (int64_t)m * nslices;
  const unsigned grid = (unsigned)((warps + 1) / 2);
  if (fuse)
    cs_gather_kernel<NV, U, true><<<grid, 64, 0, st>>>(A, n, d, m, nslices, hist, tile_sums, nchunks, perm, bvec, x,
                                                        SA, gpart, scale);
  else
    cs_gather_kernel<NV, U, false><<<grid, 64, 0, st>>>(A, n, d, m, nslices, hist, tile_sums, nchunks, perm,
                                                         nullptr, nullptr, SA, nullptr, scale);
  return cudaGetLastError();
}
}  // namespace

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
