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
constexpr size_t kTileBudget = 216 * 1024;

// v2: rows arrive through a double-buffered cp.async staging ring (R rows x
// DC columns, 16-byte pieces), so the HBM stream keeps a whole stage in flight
// while the tile is updated.  Per stage, warp w hashes the stage's rows for
// its blocks j = w, w + nw, ... into shared memory (one hash per (row, block)
// per slice), then applies the updates with lanes = (row, column): G = 32/DC
// rows x DC columns per instruction, so each row's DC contiguous doubles
// share a bank segment.  Lanes of one warp that hit the same (bucket, column)
// are serialised by match_any rank (= row order), so every tile element is a
// left-to-right sum in row order; no atomics.
constexpr int kSR = 128;  // rows per stage
template <int DC>
__global__ void __launch_bounds__(256) sjlt_dense_kernel(const double *__restrict__ A, int64_t n, int d, int m,
                                                         int s, uint64_t key, int64_t row_offset,
                                                         int64_t rows_per_split, double *__restrict__ partials) {
  extern __shared__ __align__(16) double smem[];
  double *tile = smem;                                   // m x DC
  double *stage = tile + (size_t)m * DC;                 // 2 x kSR x DC
  uint32_t *bsm = reinterpret_cast<uint32_t *>(stage + 2 * kSR * DC);  // nw x kSR (bucket | sign << 31)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int c0 = blockIdx.x * DC;
  const int dcv = min(DC, d - c0);  // valid columns of this slice
  for (int e = threadIdx.x; e < m * DC; e += blockDim.x) tile[e] = 0.0;
  const uint32_t M = (uint32_t)(m / s);
  const int64_t r0 = min(n, (int64_t)blockIdx.y * rows_per_split);
  const int64_t r1 = min(n, r0 + rows_per_split);
  const int64_t nst = (r1 - r0 + kSR - 1) / kSR;
  // 16-byte pieces per staged row when the slice is 16-byte aligned, else 8-byte
  const bool vec16 = ((DC * 8) % 16 == 0) && ((c0 * 8) % 16 == 0) && ((d * 8) % 16 == 0) && dcv == DC;
  auto issue = [&](int64_t k) {
    if (k < nst) {
      double *dst = stage + (size_t)(k & 1) * kSR * DC;
      const int64_t rb = r0 + k * kSR;
      const int rows = (int)min((int64_t)kSR, r1 - rb);
      if (vec16) {
        constexpr int P = (DC * 8) / 16;
        for (int e = threadIdx.x; e < rows * P; e += blockDim.x) {
          const int r = e / P, p = e % P;
          const unsigned sa = (unsigned)__cvta_generic_to_shared(dst + r * DC + 2 * p);
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(A + (rb + r) * d + c0 + 2 * p)
                       : "memory");
        }
      } else {
        for (int e = threadIdx.x; e < rows * DC; e += blockDim.x) {
          const int r = e / DC, c = e % DC;
          const unsigned sa = (unsigned)__cvta_generic_to_shared(dst + r * DC + c);
          const int cc = c < dcv ? c : 0;
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(A + (rb + r) * d + c0 + cc)
                       : "memory");
        }
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  issue(0);
  constexpr int G = 32 / DC;  // rows per instruction
  const int rr = lane / DC, cc = lane % DC;
  const bool lane_on = rr < G && cc < dcv;
  const unsigned lt = lanemask_lt();
  for (int64_t k = 0; k < nst; ++k) {
    issue(k + 1);
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncthreads();  // stage k visible to all; previous stage fully consumed
    const double *st = stage + (size_t)(k & 1) * kSR * DC;
    const int64_t rb = r0 + k * kSR;
    const int rows = (int)min((int64_t)kSR, r1 - rb);
    for (int j = warp; j < s; j += nw) {
      uint32_t *bj = bsm + warp * kSR;
      for (int r = lane; r < rows; r += 32) {
        bool neg;
        const uint32_t b = hash_bucket(key, (uint64_t)(row_offset + rb + r), (uint32_t)j, (uint32_t)s, M, neg);
        bj[r] = b | (neg ? 0x80000000u : 0u);
      }
      __syncwarp();
      for (int g0 = 0; g0 < rows; g0 += G) {
        const int r = g0 + rr;
        const bool on = lane_on && r < rows;
        const uint32_t be = on ? bj[r] : 0xffffffffu;
        const uint32_t b = be & 0x7fffffffu;
        double v = on ? st[r * DC + cc] : 0.0;
        if (be >> 31) v = -v;
        const uint32_t keyv = on ? b * DC + cc : 0xffffffffu;
        const unsigned mask = __match_any_sync(0xffffffffu, keyv);
        const int rank = __popc(mask & lt);
        const int maxr = __reduce_max_sync(0xffffffffu, (unsigned)(on ? rank : 0));
        for (int rd = 0; rd <= maxr; ++rd) {
          if (on && rank == rd) tile[keyv] += v;
          __syncwarp();
        }
      }
      __syncwarp();  // bj is rewritten for the next block
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  double *out = partials + (int64_t)blockIdx.y * m * d;
  for (int e = threadIdx.x; e < m * DC; e += blockDim.x) {
    const int b = e / DC, c = e - b * DC;
    if (c < dcv) out[(int64_t)b * d + c0 + c] = tile[e];
  }
}

template <int DC>
void launch_dc(const SjltPlan &p, const double *A, uint64_t key, int64_t row_offset, double *partials,
               cudaStream_t st) {
  const int threads = 32 * std::min(p.s, 8);
  const int64_t rps = (p.n + p.nsplit - 1) / p.nsplit;
  IHS_SMEM_ATTR(sjlt_dense_kernel<DC>, p.smem);
  dim3 grid(p.nslices, p.nsplit);
  sjlt_dense_kernel<DC><<<grid, threads, p.smem, st>>>(A, p.n, (int)p.d, (int)p.m, p.s, key, row_offset,
                                                       std::max<int64_t>(rps, 1), partials);
}
}  // namespace

// SA[e] = scale * sum_k partials[k][e], k ascending.
__global__ void sum_splits_kernel(const double *__restrict__ partials, int64_t count, int nsplit, double scale,
                                  double *__restrict__ SA) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x) {
    double t = 0.0;
    for (int k = 0; k < nsplit; ++k) t += partials[(int64_t)k * count + e];
    SA[e] = scale == 1.0 ? t : t * scale;
  }
}

cudaError_t launch_sum_splits(const double *partials, int64_t count, int nsplit, double scale, double *SA,
                              cudaStream_t st, LaunchCounter lc) {
  if (count <= 0) return cudaSuccess;
  const int grid = (int)std::min<int64_t>((count + 255) / 256, 148 * 8);
  sum_splits_kernel<<<grid, 256, 0, st>>>(partials, count, nsplit, scale, SA);
  lc.add();
  return cudaGetLastError();
}

bool sjlt_plan(int64_t n, int64_t d, int64_t m, int s, int num_sms, SjltPlan &p) {
  p.n = n;
  p.d = d;
  p.m = m;
  p.s = s;
  int64_t dc_max = (int64_t)(kTileBudget / (8 * (size_t)m + 2 * 128 * 8));
  if (dc_max < 1) return false;
  static const int kDC[] = {16, 8, 6, 4, 2, 1};  // DC <= 32 (lanes = rows x columns)
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
  p.smem = (size_t)m * dc * 8 + (size_t)2 * 128 * dc * 8 + (size_t)8 * 128 * 4;
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
  lc.add();
  { cudaError_t e = cudaGetLastError(); if (e != cudaSuccess) return e; }
  return launch_sum_splits(partials, p.m * p.d, p.nsplit, scale, SA, st, lc);
}

}  // namespace ihs
