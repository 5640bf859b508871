// a2 for dense A with an SJLT of s > 1 nonzeros per column, in ONE pass over A
// (s stacked independent CountSketches of m/s rows each;
// cost s * nnz(A); scaled by 1/sqrt(s)).
//
// Each CTA owns a shared-memory tile of all m sketch rows x 4 columns of A and
// streams a contiguous row range of that 4-column slice once (cp.async,
// double-buffered stages of kSR rows).  Two warps per SJLT block j, one per
// column pair: the s updates of a row land in disjoint bucket ranges
// [j M, (j+1) M) and the two warps of a block own disjoint columns, so no two
// warps touch the same tile element and no atomics are needed (fp64 shared
// atomics are CAS loops on sm_100a).  Rows of one 16-row window that share a
// bucket are applied in rank (= row) order, so every tile element is a
// left-to-right sum over the slice's rows.  Row-range partials are summed in
// a fixed order and scaled once (sum_splits).
//
// Bound: shared memory.  Every element costs s fp64 read-modify-writes at
// random buckets (B200, tools/probe: 3.4 random vs 7.3 conflict-free updates
// per clock per SM) plus s conflict-free stage reads.
#include "common.cuh"
#include "kernels.h"

namespace ihs {

namespace {
constexpr int kSW = 4;    // columns per CTA slice (two column pairs)
constexpr int kSR = 512;  // rows per stage

// Warp w = 2 j + h applies SJLT block j to column pair h of the slice (16
// warps for s = 8).  Tile and stage are column-pair-major (double2 per bucket
// / row), so 8 consecutive stage rows are 128 contiguous bytes.  Lanes = 16
// rows x 2 columns.
//   hash pass (lanes = rows; the block's two warps take alternate 32-row
//     chunks): bucket | sign for block j, plus each row's rank among the rows
//     of its 16-row apply window with the same bucket and the window's largest
//     rank (xor-shuffles within 16-lane segments);
//   apply: one read-modify-write per lane per window, in rank order when a
//     bucket repeats in the window (probability ~120/M).
__global__ void __launch_bounds__(1024, 1) sjlt_stream_kernel(const double *__restrict__ A, int64_t n, int d, int m,
                                                              int s, uint32_t M, uint64_t key, int64_t row_offset,
                                                              int64_t rows_per_split, double *__restrict__ partials) {
  extern __shared__ __align__(16) double smem[];
  double *tile = smem;                                                 // [2 pair][m][2]
  double *stage = tile + (size_t)m * kSW;                              // [2 buf][2 pair][kSR][2]
  uint32_t *hb = reinterpret_cast<uint32_t *>(stage + 2 * kSR * kSW);  // [s][kSR]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int j = warp >> 1, h = warp & 1;  // SJLT block, column pair
  const int q = lane >> 1, c = lane & 1;  // row in window, column in pair
  const int c0 = blockIdx.x * kSW;
  const int dcv = min(kSW, d - c0);
  for (int e = threadIdx.x; e < m * kSW; e += blockDim.x) tile[e] = 0.0;
  const int64_t r0 = min(n, (int64_t)blockIdx.y * rows_per_split);
  const int64_t r1 = min(n, r0 + rows_per_split);
  const int64_t nst = (r1 - r0 + kSR - 1) / kSR;
  const bool vec16 = (d % 2 == 0) && dcv == kSW;  // 16-byte pieces (c0 is a multiple of 4)
  auto issue = [&](int64_t k) {
    if (k < nst) {
      double *dst = stage + (size_t)(k & 1) * kSR * kSW;
      const int64_t rb = r0 + k * kSR;
      const int rows = (int)min((int64_t)kSR, r1 - rb);
      if (vec16) {
        for (int e = threadIdx.x; e < rows * 2; e += blockDim.x) {
          const int r = e >> 1, p = e & 1;
          const unsigned sa = (unsigned)__cvta_generic_to_shared(dst + ((size_t)p * kSR + r) * 2);
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(A + (rb + r) * d + c0 + 2 * p)
                       : "memory");
        }
      } else {
        for (int e = threadIdx.x; e < rows * kSW; e += blockDim.x) {
          const int r = e >> 2, cc = e & 3;
          const unsigned sa = (unsigned)__cvta_generic_to_shared(dst + ((size_t)(cc >> 1) * kSR + r) * 2 + (cc & 1));
          const int sz = cc < dcv ? 8 : 0;  // zero-fill the columns past d
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(sa),
                       "l"(A + (rb + r) * d + c0 + (cc < dcv ? cc : 0)), "r"(sz)
                       : "memory");
        }
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  issue(0);
  uint32_t *hbj = hb + j * kSR;
  double *tj = tile + (size_t)h * m * 2;
  for (int64_t k = 0; k < nst; ++k) {
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();  // stage k landed for everyone; stage k-1 fully consumed
    issue(k + 1);
    const int64_t rb = r0 + k * kSR;
    const int rows = (int)min((int64_t)kSR, r1 - rb);
    for (int r = 32 * h + lane; r - lane < rows; r += 64) {
      bool neg = false;
      uint32_t b = 0x800000u + lane;  // rows past the end: distinct dummies
      if (r < rows) b = hash_bucket(key, (uint64_t)(row_offset + rb + r), (uint32_t)j, (uint32_t)s, M, neg);
      uint32_t rank = 0;
#pragma unroll
      for (int x = 1; x < 16; ++x) {
        const uint32_t o = __shfl_xor_sync(0xffffffffu, b, x);
        rank += (o == b && (lane ^ x) < lane) ? 1u : 0u;
      }
      uint32_t wmax = rank;
#pragma unroll
      for (int x = 1; x < 16; x <<= 1) wmax = max(wmax, __shfl_xor_sync(0xffffffffu, wmax, x));
      if (r < rows) hbj[r] = b | (rank << 23) | (wmax << 27) | (neg ? 0x80000000u : 0u);
    }
    __syncthreads();  // hb of the stage complete
    // entry bits: 0-22 bucket, 23-26 rank, 27-30 window max rank, 31 sign
    const double *st = stage + (size_t)(k & 1) * kSR * kSW + (size_t)h * kSR * 2;
    uint32_t en = q < rows ? hbj[q] : 0xffffffffu;
    double vn = q < rows ? st[q * 2 + c] : 0.0;
    for (int g0 = 0; g0 < rows; g0 += 16) {
      const uint32_t e = en;
      const double v0 = vn;
      const int rn = g0 + 16 + q;  // prefetch the next window
      en = rn < rows ? hbj[rn] : 0xffffffffu;
      vn = rn < rows ? st[rn * 2 + c] : 0.0;
      const bool on = e != 0xffffffffu;
      const double v = (e >> 31) ? -v0 : v0;
      double *t = tj + (size_t)(e & 0x7fffffu) * 2 + c;
      const uint32_t wmax = __shfl_sync(0xffffffffu, (e >> 27) & 15u, 0);  // the window's rows share it
      if (wmax == 0) {
        if (on) *t += v;
      } else {
        const uint32_t rank = (e >> 23) & 15u;
        for (uint32_t rd = 0; rd <= wmax; ++rd) {
          if (on && rank == rd) *t += v;
          __syncwarp();
        }
      }
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  double *out = partials + (int64_t)blockIdx.y * m * d;
  for (int e = threadIdx.x; e < m * kSW; e += blockDim.x) {
    const int b = e >> 2, cc = e & 3;
    if (cc < dcv) out[(int64_t)b * d + c0 + cc] = tile[((size_t)(cc >> 1) * m + b) * 2 + (cc & 1)];
  }
}
}  // namespace

bool sjlt_stream_plan(int64_t n, int64_t d, int64_t m, int s, int num_sms, SjltPlan &p) {
  if (s < 2 || s > 16 || m % s != 0 || m >= (1 << 23)) return false;
  p.n = n;
  p.d = d;
  p.m = m;
  p.s = s;
  p.dc = kSW;
  p.smem = (size_t)m * kSW * 8 + (size_t)2 * kSR * kSW * 8 + (size_t)s * kSR * 4;
  if (p.smem > 220 * 1024) return false;
  p.nslices = (int)((d + kSW - 1) / kSW);
  const int per_sm = std::max(1, (int)((227 * 1024) / (p.smem + 1024)));
  // about one wave of CTAs: nslices x nsplit ~ num_sms * per_sm
  int64_t ns = std::max<int64_t>(1, ((int64_t)num_sms * per_sm) / p.nslices);
  ns = std::min<int64_t>(ns, std::max<int64_t>(1, (n + kSR - 1) / kSR));
  p.nsplit = (int)ns;
  return true;
}

cudaError_t launch_sjlt_stream(const SjltPlan &p, const double *A, uint64_t key, int64_t row_offset,
                               double *partials, double *SA, double scale, cudaStream_t st, LaunchCounter lc) {
  IHS_SMEM_ATTR(sjlt_stream_kernel, p.smem);
  const int64_t rps = (p.n + p.nsplit - 1) / p.nsplit;
  dim3 grid(p.nslices, p.nsplit);
  sjlt_stream_kernel<<<grid, 64 * p.s, p.smem, st>>>(A, p.n, (int)p.d, (int)p.m, p.s, (uint32_t)(p.m / p.s), key,
                                                     row_offset, std::max<int64_t>(rps, 1), partials);
  lc.add();
  return launch_sum_splits(partials, p.m * p.d, p.nsplit, scale, SA, st, lc);
}

}  // namespace ihs
