// a2 for dense A with an SJLT of s > 1 nonzeros per column (PAPER.md:180-184:
// s stacked independent CountSketches of m/s rows; cost s * nnz(A),
// PAPER.md:238-240; scaled by 1/sqrt(s)).
//
// Each CTA owns a shared-memory tile of ALL m sketch rows x DC columns and
// streams a contiguous row range of A once; warp j applies block j, so the s
// updates of a row land in disjoint bucket ranges (no cross-warp conflicts;
// fp64 smem atomics are CAS loops on sm_100a, so none are used).  Lanes are
// rows; lanes of one warp that share a bucket are serialised in rank (= row)
// order with match_any, so every tile element is a left-to-right sum in row
// order.  Row-range partials are summed in a fixed order and scaled once.
// On-chip (shared-memory) bandwidth bound: s read-modify-writes per element.
#include "common.cuh"
#include "kernels.h"

namespace ihs {

namespace {
constexpr size_t kTileBudget = 200 * 1024;

template <int DC>
__global__ void __launch_bounds__(512) sjlt_dense_kernel(const double *__restrict__ A, int64_t n, int d, int m,
                                                         int s, uint64_t key, int64_t row_offset,
                                                         int64_t rows_per_split, double *__restrict__ partials) {
  extern __shared__ double tile[];  // m x DC, bucket-major
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int c0 = blockIdx.x * DC;
  for (int e = threadIdx.x; e < m * DC; e += blockDim.x) tile[e] = 0.0;
  __syncthreads();
  const uint32_t M = (uint32_t)(m / s);
  const int64_t r0 = min(n, (int64_t)blockIdx.y * rows_per_split);
  const int64_t r1 = min(n, r0 + rows_per_split);
  const unsigned lt = lanemask_lt();
  bool cval[DC];
#pragma unroll
  for (int c = 0; c < DC; ++c) cval[c] = c0 + c < d;
  for (int j = warp; j < s; j += nwarps) {
    for (int64_t base = r0; base < r1; base += 32) {
      const int64_t r = base + lane;
      const bool valid = r < r1;
      bool neg = false;
      const uint32_t b = valid ? hash_bucket(key, (uint64_t)(row_offset + r), (uint32_t)j, (uint32_t)s, M, neg)
                               : 0xffffffffu;
      double v[DC];
      const double *rowp = A + (valid ? r : 0) * d + c0;
#pragma unroll
      for (int c = 0; c < DC; ++c) {
        double a = (valid && cval[c]) ? __ldg(rowp + c) : 0.0;
        v[c] = neg ? -a : a;
      }
      const unsigned mask = __match_any_sync(0xffffffffu, b);
      const int rank = __popc(mask & lt);
      const int maxr = __reduce_max_sync(0xffffffffu, (unsigned)rank);
      for (int rd = 0; rd <= maxr; ++rd) {
        if (valid && rank == rd) {
          double *t = tile + (size_t)b * DC;
#pragma unroll
          for (int c = 0; c < DC; ++c) t[c] += v[c];
        }
        __syncwarp();
      }
    }
  }
  __syncthreads();
  double *out = partials + (int64_t)blockIdx.y * m * d;
  for (int e = threadIdx.x; e < m * DC; e += blockDim.x) {
    const int b = e / DC, c = e - b * DC;
    if (c0 + c < d) out[(int64_t)b * d + c0 + c] = tile[e];
  }
}

// SA[e] = scale * sum_k partials[k][e], k ascending.
__global__ void sum_splits_kernel(const double *__restrict__ partials, int64_t count, int nsplit, double scale,
                                  double *__restrict__ SA) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x) {
    double t = 0.0;
    for (int k = 0; k < nsplit; ++k) t += partials[(int64_t)k * count + e];
    SA[e] = scale == 1.0 ? t : t * scale;
  }
}

template <int DC>
void launch_dc(const SjltPlan &p, const double *A, uint64_t key, int64_t row_offset, double *partials,
               cudaStream_t st) {
  const int threads = 32 * std::min(p.s, 16);
  const int64_t rps = (p.n + p.nsplit - 1) / p.nsplit;
  IHS_SMEM_ATTR(sjlt_dense_kernel<DC>, p.smem);
  dim3 grid(p.nslices, p.nsplit);
  sjlt_dense_kernel<DC><<<grid, threads, p.smem, st>>>(A, p.n, (int)p.d, (int)p.m, p.s, key, row_offset,
                                                       std::max<int64_t>(rps, 1), partials);
}
}  // namespace

bool sjlt_plan(int64_t n, int64_t d, int64_t m, int s, int num_sms, SjltPlan &p) {
  p.n = n;
  p.d = d;
  p.m = m;
  p.s = s;
  int64_t dc_max = (int64_t)(kTileBudget / (8 * (size_t)m));
  if (dc_max < 1) return false;
  static const int kDC[] = {16, 8, 6, 4, 2, 1};
  int dc = 1;
  for (int c : kDC)
    if (c <= dc_max && (c <= d || c == 1)) {
      dc = c;
      break;
    }
  // prefer the smallest template that still covers d in one slice
  if (d < dc) {
    for (int c : kDC)
      if (c >= d && c <= dc_max) dc = c;
  }
  p.dc = dc;
  p.nslices = (int)((d + dc - 1) / dc);
  p.smem = (size_t)m * dc * 8;
  int blocks_per_sm = std::max<int>(1, (int)((227 * 1024) / (p.smem + 1024)));
  blocks_per_sm = std::min(blocks_per_sm, 4);
  int64_t want = (int64_t)num_sms * blocks_per_sm * 4;
  int64_t ns = std::max<int64_t>(1, (want + p.nslices - 1) / p.nslices);
  ns = std::min<int64_t>(ns, std::max<int64_t>(1, n / 1024));
  p.nsplit = (int)ns;
  return true;
}

cudaError_t launch_sjlt_dense(const SjltPlan &p, const double *A, uint64_t key, int64_t row_offset, double *partials,
                              double *SA, double scale, cudaStream_t st, LaunchCounter lc) {
  switch (p.dc) {
    case 16: launch_dc<16>(p, A, key, row_offset, partials, st); break;
    case 8: launch_dc<8>(p, A, key, row_offset, partials, st); break;
    case 6: launch_dc<6>(p, A, key, row_offset, partials, st); break;
    case 4: launch_dc<4>(p, A, key, row_offset, partials, st); break;
    case 2: launch_dc<2>(p, A, key, row_offset, partials, st); break;
    default: launch_dc<1>(p, A, key, row_offset, partials, st); break;
  }
  const int64_t count = p.m * p.d;
  int grid = (int)std::min<int64_t>((count + 255) / 256, 148 * 8);
  sum_splits_kernel<<<grid, 256, 0, st>>>(partials, count, p.nsplit, scale, SA);
  lc.add(2);
  return cudaGetLastError();
}

}  // namespace ihs
