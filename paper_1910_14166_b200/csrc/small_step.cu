// One IHS iteration (a1-a6, OLS) for a small dense problem in ONE launch of
// one CTA (BASELINE.json configs[0]: 2000 x 10, m = 200).  At this size every
// kernel of the general path runs for a few microseconds and the step is the
// sum of launch latencies (r01: 0.059 ms per step over 7 launches); here the
// whole iteration is phases of one 512-thread CTA separated by __syncthreads:
//   1. residuals r_i = b_i - a_i . x and the s bucket codes of every row
//      (hash of reading R1, global rows), kept in shared memory;
//   2. per SJLT block, a stable counting sort of the rows by bucket (one warp
//      per block: counts, scan, ballot-ranked placement in ascending rows);
//   3. SA[b][c] = sum over bucket b's rows in ascending order of +-A[row][c]
//      (the oracle's order: bit-identical for CountSketch), x 1/sqrt(s);
//   4. g[c] = sum_i A[i][c] r_i from 32 fixed row slices added in order;
//   5. H = SA^T SA (d x d);  6. Cholesky of H (one warp, d <= 32), L y = g,
//      L^T u = y, x_next = x + u (Eq. (2)); a pivot <= 0 sets
//      IHS_ERR_NOT_SPD and leaves x_next = x (reading R13).
// Limits: d <= 32, s <= 32, n * (8 + 2 s) + m * d * 8 + ... within 200 KB.
#include "common.cuh"
#include "kernels.h"
#include "chol_blocks.cuh"

namespace ihs {

namespace {
constexpr int kThreads = 512;
constexpr int kSlices = 32;

__global__ void __launch_bounds__(kThreads) small_step_kernel(const double *__restrict__ A, int n, int d,
                                                              const double *__restrict__ bvec,
                                                              const double *__restrict__ x, uint64_t key,
                                                              int64_t row_offset, int s, int M, double scale,
                                                              double *__restrict__ x_next, double *SA_out,
                                                              double *g_out, double *H_out, int *status) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int m = M * s;
  double *r = reinterpret_cast<double *>(smem_raw);        // n
  double *SA = r + n;                                      // m x d
  double *gp = SA + (size_t)m * d;                         // kSlices x d
  double *H = gp + kSlices * d;                            // 32 x 33 (padded)
  double *xs = H + 32 * 33;                                // 32
  double *misc = xs + 32;                                  // 64 (Cholesky column buffer) + 32 (rd)
  uint16_t *code = reinterpret_cast<uint16_t *>(misc + 96);          // s x n: bucket | neg << 15
  uint16_t *ent = code + (size_t)s * n;                              // s x n: rows sorted by bucket
  int32_t *cnt = reinterpret_cast<int32_t *>(ent + (size_t)s * n + ((s * n) & 1));  // s x (M + 1)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < 32) xs[tid] = tid < d ? x[tid] : 0.0;
  for (int e = tid; e < s * (M + 1); e += kThreads) cnt[e] = 0;
  __syncthreads();
  // 1. residuals and codes
  for (int i = tid; i < n; i += kThreads) {
    const double *ai = A + (size_t)i * d;
    double dot = 0.0;
    for (int c = 0; c < d; ++c) dot = fma(ai[c], xs[c], dot);
    r[i] = bvec[i] - dot;
    for (int j = 0; j < s; ++j) {
      bool neg;
      const uint32_t b = hash_bucket(key, (uint64_t)(row_offset + i), (uint32_t)j, (uint32_t)s, (uint32_t)M, neg) -
                         (uint32_t)j * (uint32_t)M;
      code[(size_t)j * n + i] = (uint16_t)(b | (neg ? 0x8000u : 0u));
      atomicAdd(&cnt[j * (M + 1) + b], 1);
    }
  }
  __syncthreads();
  // 2. per block (one warp each): exclusive scan, then stable placement
  for (int j = warp; j < s; j += kThreads / 32) {
    int32_t *ct = cnt + j * (M + 1);
    int carry = 0;
    for (int b0 = 0; b0 < M; b0 += 32) {
      const int b = b0 + lane;
      const int v = b < M ? ct[b] : 0;
      int incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (b < M) ct[b] = carry + incl - v;
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) ct[M] = carry;
    __syncwarp();
    const uint16_t *cd = code + (size_t)j * n;
    uint16_t *en = ent + (size_t)j * n;
    const int nbits = M > 1 ? 32 - __clz(M - 1) : 1;
    for (int rb = 0; rb < n; rb += 32) {
      const int i = rb + lane;
      const bool v = i < n;
      const uint32_t b = v ? (cd[i] & 0x7fffu) : 0u;
      const unsigned peers = peers_by_ballot(b, nbits, v);
      const int rank = __popc(peers & lanemask_lt());
      int base = 0;
      if (v) base = ct[b];
      __syncwarp();
      if (v) {
        en[base + rank] = (uint16_t)i;
        if (rank == 0) ct[b] = base + __popc(peers);
      }
      __syncwarp();
    }
  }
  __syncthreads();
  // 3. bucket sums in ascending row order (ct[b] now holds the END of bucket b)
  for (int e = tid; e < m * d; e += kThreads) {
    const int bb = e / d, c = e - bb * d;
    const int j = bb / M, b = bb - j * M;
    const int32_t *ct = cnt + j * (M + 1);
    const int end = ct[b], beg = b > 0 ? ct[b - 1] : 0;
    const uint16_t *en = ent + (size_t)j * n;
    const uint16_t *cd = code + (size_t)j * n;
    double acc = 0.0;
    for (int k = beg; k < end; ++k) {
      const int i = en[k];
      acc = fma((cd[i] & 0x8000u) ? -1.0 : 1.0, A[(size_t)i * d + c], acc);
    }
    SA[e] = scale == 1.0 ? acc : acc * scale;
  }
  // 4. gradient slices
  for (int e = tid; e < kSlices * d; e += kThreads) {
    const int sl = e / d, c = e - sl * d;
    const int i0 = (int)((int64_t)n * sl / kSlices), i1 = (int)((int64_t)n * (sl + 1) / kSlices);
    double acc = 0.0;
    for (int i = i0; i < i1; ++i) acc = fma(A[(size_t)i * d + c], r[i], acc);
    gp[e] = acc;
  }
  __syncthreads();
  // 5. H = SA^T SA and g
  for (int e = tid; e < d * d; e += kThreads) {
    const int p = e / d, q = e - p * d;
    double acc = 0.0;
    for (int bb = 0; bb < m; ++bb) acc = fma(SA[bb * d + p], SA[bb * d + q], acc);
    H[p * 33 + q] = acc;
  }
  double *gv = misc + 64;  // 32 (reuses the rd slot until the factorisation)
  if (tid < d) {
    double acc = 0.0;
    for (int sl = 0; sl < kSlices; ++sl) acc += gp[sl * d + tid];
    gv[tid] = acc;
  }
  __syncthreads();
  if (H_out)
    for (int e = tid; e < d * d; e += kThreads) H_out[e] = H[(e / d) * 33 + e % d];
  if (SA_out)
    for (int e = tid; e < m * d; e += kThreads) SA_out[e] = SA[e];
  if (g_out && tid < d) g_out[tid] = gv[tid];
  __syncthreads();  // (H_out, gv read above before warp 0 rewrites them)
  // 6. Cholesky + solves (warp 0): pad H to 32 x 32 with the identity
  if (warp == 0) {
    for (int c = d; c < 32; ++c) H[lane * 33 + c] = (lane == c) ? 1.0 : 0.0;
    for (int rr = d; rr < 32; ++rr) H[rr * 33 + lane] = (lane == rr) ? 1.0 : 0.0;
    __syncwarp();
    double gl = lane < d ? gv[lane] : 0.0;
    __syncwarp();
    double *rdv = misc + 64;  // reciprocal pivots (g already in registers)
    const bool bad = warp_chol32(H, 33, rdv, d, misc);
    __syncwarp();  // row k of L (lane k's stores) and rd (lane 0's) are read by every lane below
    if (bad) {
      if (lane < d) x_next[lane] = xs[lane];
      if (lane == 0) set_status(status, 3 /* IHS_ERR_NOT_SPD */);
    } else {
      // forward L y = g, then back L^T u = y: lane k holds y_k / u_k; the
      // pivot of step k is lane k's own 1/L_kk, applied before the broadcast
      const double rdl = rdv[lane];
      double y = gl;
      for (int k = 0; k < d; ++k) {
        const double yk = __shfl_sync(0xffffffffu, y * rdl, k);
        if (lane == k) y = yk;
        if (lane > k) y = fma(-H[lane * 33 + k], yk, y);
      }
      double u = y;
      for (int k = d - 1; k >= 0; --k) {
        const double uk = __shfl_sync(0xffffffffu, u * rdl, k);
        if (lane == k) u = uk;
        if (lane < k) u = fma(-H[k * 33 + lane], uk, u);
      }
      if (lane < d) x_next[lane] = xs[lane] + u;
    }
  }
}
}  // namespace

size_t small_step_smem(int64_t n, int64_t d, int64_t m, int s) {
  const int64_t M = m / s;
  return (size_t)(n + m * d + kSlices * d + 32 * 33 + 32 + 96) * 8 + (size_t)(2 * s * n + 2) * 2 +
         (size_t)s * (M + 1) * 4 + 16;
}

bool small_step_supported(int64_t n, int64_t d, int64_t m, int s) {
  return n >= 1 && n <= 32768 && d >= 1 && d <= 32 && s >= 1 && s <= 32 && m % s == 0 && m / s <= 32768 &&
         small_step_smem(n, d, m, s) <= 200 * 1024;
}

cudaError_t launch_small_step(const double *A, int64_t n, int64_t d, const double *b, const double *x, uint64_t key,
                              int64_t row_offset, int64_t m, int s, double scale, double *x_next, double *SA_out,
                              double *g_out, double *H_out, int *status, cudaStream_t st, LaunchCounter lc) {
  const size_t smem = small_step_smem(n, d, m, s);
  IHS_SMEM_ATTR(small_step_kernel, smem);
  small_step_kernel<<<1, kThreads, smem, st>>>(A, (int)n, (int)d, b, x, key, row_offset, s, (int)(m / s), scale,
                                               x_next, SA_out, g_out, H_out, status);
  lc.add();
  return cudaGetLastError();
}

}  // namespace ihs
