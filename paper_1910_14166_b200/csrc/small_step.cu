// One IHS iteration (a1-a6, OLS) for a small dense problem in ONE launch of
// one CTA (BASELINE.json configs[0]: 2000 x 10, m = 200).  At this size every
// kernel of the general path runs for a few microseconds and the step is the
// sum of launch latencies (r01: 0.059 ms per step over 7 launches); here the
// whole iteration is phases of one 512-thread CTA separated by __syncthreads,
// on A staged once in shared memory (coalesced, loads in flight):
//   1. residuals r_i = b_i - a_i . x and the s bucket codes of every row
//      (hash of reading R1, global rows);
//   2. per SJLT block, a stable counting sort of the rows by bucket: sort warp
//      w counts its contiguous row range, a scan over (block, bucket, warp)
//      gives every warp its base per bucket, and each warp places its rows 32
//      at a time (ballot ranks) -- ascending rows within every bucket;
//   3. SA[b][c] = sum over bucket b's rows in ascending order of +-A[row][c]
//      (the oracle's order: bit-identical for CountSketch), x 1/sqrt(s);
//   4. g[c] = sum_i A[i][c] r_i from 32 fixed row slices added in order;
//   5. H = SA^T SA (d x d, four fixed partial sums per entry);
//   6. Cholesky of H with row i in registers of lane i of warp 0 (d column
//      steps), L y = g, L^T u = y, x_next = x + u (Eq. (2)); a
//      pivot <= 0 sets IHS_ERR_NOT_SPD and leaves x_next = x (reading R13).
// (A first version that read A from global memory in every phase, sorted in
// one warp per block and padded the Cholesky to 32 columns took 46 us per
// iteration for C1.)
#include "common.cuh"
#include "kernels.h"

namespace ihs {

namespace {
constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kSortWarps = 8;
constexpr int kSlices = 32;
constexpr int kHParts = 4;

struct SmallLayout {
  size_t A, r, SA, gp, Hp, H, xs, col, code, ent, cnt, total;
};
__host__ __device__ inline SmallLayout small_layout(int n, int d, int M, int s) {
  SmallLayout L;
  const int m = M * s;
  size_t o = 0;
  L.A = o;    o += (size_t)n * d * 8;
  L.r = o;    o += (size_t)n * 8;
  L.SA = o;   o += (size_t)m * d * 8;
  L.gp = o;   o += (size_t)kSlices * d * 8;
  L.Hp = o;   o += (size_t)kHParts * d * d * 8;
  L.H = o;    o += (size_t)d * 33 * 8;
  L.xs = o;   o += 32 * 8;
  L.col = o;  o += 64 * 8;  // column-broadcast slots of the factorisation
  L.code = o; o += (size_t)s * n * 2;
  L.ent = o;  o += (size_t)s * n * 2;
  o = (o + 3) & ~(size_t)3;
  L.cnt = o;  o += (size_t)s * M * kSortWarps * 4;  // per (block, bucket, sort warp): counts -> offsets
  L.total = o + 16;
  return L;
}

// T iterations in one launch: A is staged once; iteration t uses the key of
// iteration iter0 + t, starts from x^t (x for t = 0) and writes x^{t+1} to
// xout + t d.  (One launch per iteration re-staged A from L2 and paid the
// launch gap each time.)
__global__ void __launch_bounds__(kThreads) small_step_kernel(const double *__restrict__ A, int n, int d,
                                                              const double *__restrict__ bvec,
                                                              const double *__restrict__ x, uint64_t seed,
                                                              uint64_t iter0, int T, int64_t row_offset, int s, int M,
                                                              double scale, double *__restrict__ xout, double *SA_out,
                                                              double *g_out, double *H_out, int *status) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int wsum[kWarps];
  const SmallLayout Ly = small_layout(n, d, M, s);
  double *As = reinterpret_cast<double *>(smem_raw + Ly.A);
  double *r = reinterpret_cast<double *>(smem_raw + Ly.r);
  double *SA = reinterpret_cast<double *>(smem_raw + Ly.SA);
  double *gp = reinterpret_cast<double *>(smem_raw + Ly.gp);
  double *Hp = reinterpret_cast<double *>(smem_raw + Ly.Hp);
  double *H = reinterpret_cast<double *>(smem_raw + Ly.H);
  double *xs = reinterpret_cast<double *>(smem_raw + Ly.xs);
  double *colb = reinterpret_cast<double *>(smem_raw + Ly.col);
  uint16_t *code = reinterpret_cast<uint16_t *>(smem_raw + Ly.code);  // [s][n]: bucket | neg << 15
  uint16_t *ent = reinterpret_cast<uint16_t *>(smem_raw + Ly.ent);    // [s][n]: rows sorted by bucket
  int32_t *cnt = reinterpret_cast<int32_t *>(smem_raw + Ly.cnt);      // [s][M][kSortWarps]
  const int m = M * s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // 0. stage A (coalesced, 8 loads in flight per thread) and x; clear the counts
  const int nd = n * d;
  for (int e0 = tid; e0 < nd; e0 += 8 * kThreads) {
    double v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int e = e0 + k * kThreads;
      v[k] = e < nd ? A[e] : 0.0;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int e = e0 + k * kThreads;
      if (e < nd) As[e] = v[k];
    }
  }
  if (tid < 32) xs[tid] = tid < d ? x[tid] : 0.0;
  for (int t = 0; t < T; ++t) {
  const uint64_t key = iter_key(seed, iter0 + (uint64_t)t);
  double *x_next = xout + (size_t)t * d;
  for (int e = tid; e < s * M * kSortWarps; e += kThreads) cnt[e] = 0;
  __syncthreads();
  // 1. residuals and codes (thread per row); counts per sort warp's row range
  for (int i = tid; i < n; i += kThreads) {
    const double *ai = As + (size_t)i * d;
    double dot = 0.0;
    for (int c = 0; c < d; ++c) dot = fma(ai[c], xs[c], dot);
    r[i] = bvec[i] - dot;
    const int sw = (int)(((int64_t)i * kSortWarps) / n);  // the sort warp owning row i (contiguous ranges)
    for (int j = 0; j < s; ++j) {
      bool neg;
      const uint32_t b = hash_bucket(key, (uint64_t)(row_offset + i), (uint32_t)j, (uint32_t)s, (uint32_t)M, neg) -
                         (uint32_t)j * (uint32_t)M;
      code[(size_t)j * n + i] = (uint16_t)(b | (neg ? 0x8000u : 0u));
      atomicAdd(&cnt[((size_t)j * M + b) * kSortWarps + sw], 1);
    }
  }
  __syncthreads();
  // 2a. exclusive scan over (block, bucket, sort warp) in that order: warp w's
  // base in bucket b follows every lower warp's rows of b (block j's entries
  // occupy [j n, (j+1) n))
  {
    const int E = s * M * kSortWarps;
    const int per = (E + kThreads - 1) / kThreads;
    const int e0 = min(E, tid * per), e1 = min(E, e0 + per);
    int loc = 0;
    for (int e = e0; e < e1; ++e) loc += cnt[e];
    int incl = loc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    int run = incl - loc;
    for (int w = 0; w < warp; ++w) run += wsum[w];
    for (int e = e0; e < e1; ++e) {
      const int c = cnt[e];
      cnt[e] = run;
      run += c;
    }
  }
  __syncthreads();
  // 2b. stable placement by the sort warps, their rows in order, 32 at a time
  if (warp < kSortWarps) {
    const int w0 = (int)(((int64_t)n * warp + kSortWarps - 1) / kSortWarps);
    const int w1 = (int)(((int64_t)n * (warp + 1) + kSortWarps - 1) / kSortWarps);
    const int nbits = M > 1 ? 32 - __clz(M - 1) : 1;
    for (int j = 0; j < s; ++j) {
      const uint16_t *cd = code + (size_t)j * n;
      int32_t *ct = cnt + (size_t)j * M * kSortWarps;
      for (int rb = w0; rb < w1; rb += 32) {
        const int i = rb + lane;
        const bool v = i < w1;
        const uint32_t b = v ? (cd[i] & 0x7fffu) : 0u;
        const unsigned peers = peers_by_ballot(b, nbits, v);
        const int rank = __popc(peers & lanemask_lt());
        int base = 0;
        if (v) base = ct[b * kSortWarps + warp];
        __syncwarp();
        if (v) {
          ent[base + rank] = (uint16_t)i;
          if (rank == 0) ct[b * kSortWarps + warp] = base + __popc(peers);
        }
        __syncwarp();
      }
    }
  }
  __syncthreads();
  // 3. bucket sums in ascending row order: bucket bb ends at the last sort
  // warp's slot, starts where the previous bucket of its block ends
  for (int e = tid; e < m * d; e += kThreads) {
    const int bb = e / d, c = e - bb * d;
    const int end = cnt[(size_t)bb * kSortWarps + kSortWarps - 1];
    const int beg = bb % M == 0 ? (bb / M) * n : cnt[(size_t)(bb - 1) * kSortWarps + kSortWarps - 1];
    const uint16_t *cd = code + (size_t)(bb / M) * n;
    double acc = 0.0;
    for (int k = beg; k < end; ++k) {
      const int i = ent[k];
      acc = fma((cd[i] & 0x8000u) ? -1.0 : 1.0, As[(size_t)i * d + c], acc);
    }
    SA[e] = scale == 1.0 ? acc : acc * scale;
  }
  // 4. gradient slices (fixed row ranges)
  for (int e = tid; e < kSlices * d; e += kThreads) {
    const int sl = e / d, c = e - sl * d;
    const int i0 = (int)((int64_t)n * sl / kSlices), i1 = (int)((int64_t)n * (sl + 1) / kSlices);
    double a0 = 0.0, a1 = 0.0;
    int i = i0;
    for (; i + 1 < i1; i += 2) {
      a0 = fma(As[(size_t)i * d + c], r[i], a0);
      a1 = fma(As[(size_t)(i + 1) * d + c], r[i + 1], a1);
    }
    if (i < i1) a0 = fma(As[(size_t)i * d + c], r[i], a0);
    gp[e] = a0 + a1;
  }
  __syncthreads();
  // 5. H = SA^T SA: kHParts fixed bucket ranges per entry, added in order
  for (int e = tid; e < kHParts * d * d; e += kThreads) {
    const int part = e / (d * d), pq = e - part * d * d;
    const int p = pq / d, q = pq - p * d;
    const int b0 = m * part / kHParts, b1 = m * (part + 1) / kHParts;
    double a0 = 0.0, a1 = 0.0;
    int bb = b0;
    for (; bb + 1 < b1; bb += 2) {
      a0 = fma(SA[bb * d + p], SA[bb * d + q], a0);
      a1 = fma(SA[(bb + 1) * d + p], SA[(bb + 1) * d + q], a1);
    }
    if (bb < b1) a0 = fma(SA[bb * d + p], SA[bb * d + q], a0);
    Hp[e] = a0 + a1;
  }
  __syncthreads();
  for (int e = tid; e < d * d; e += kThreads) {
    double acc = Hp[e];
#pragma unroll
    for (int part = 1; part < kHParts; ++part) acc += Hp[part * d * d + e];
    H[(e / d) * 33 + e % d] = acc;
    if (H_out) H_out[e] = acc;
  }
  double gl = 0.0;
  if (warp == 0 && lane < d) {
    for (int sl = 0; sl < kSlices; ++sl) gl += gp[sl * d + lane];
    if (g_out) g_out[lane] = gl;
  }
  if (SA_out)
    for (int e = tid; e < m * d; e += kThreads) SA_out[e] = SA[e];
  __syncthreads();
  if (warp == 0) {
  // 6. Cholesky: lane i holds row i of H (lower part) in registers
  double row[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) row[c] = (lane < d && c <= lane) ? H[lane * 33 + c] : 0.0;
  bool bad = false;
  double rdl = 1.0;  // this lane's 1 / L_ii
#pragma unroll
  for (int J = 0; J < 32; ++J) {
    if (J < d) {
      const double piv = __shfl_sync(0xffffffffu, row[J], J);
      bad |= !(piv > 0.0);
      double ljj, rj;
      pivot_rsqrt(piv, ljj, rj);
      const double lij = (lane > J) ? row[J] * rj : (lane == J ? ljj : 0.0);
      if (lane == J) rdl = rj;
      row[J] = lij;
      colb[(J & 1) * 32 + lane] = lij;
      __syncwarp();
#pragma unroll
      for (int k = J + 1; k < 32; ++k) row[k] = fma(-lij, colb[(J & 1) * 32 + k], row[k]);
    }
  }
  if (__any_sync(0xffffffffu, bad)) {  // x^{t+1} = x^t (the oracle's verdict, R13)
    if (lane < d) x_next[lane] = xs[lane];
    if (lane == 0) set_status(status, 3 /* IHS_ERR_NOT_SPD */);
  } else {
  // forward L y = g (lane k finishes y_k; lanes below use L[lane][k] = row[k]);
  // the pivot reciprocal is the finishing lane's own
  double y = gl;
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    if (k < d) {
      const double yk = __shfl_sync(0xffffffffu, y * rdl, k);
      if (lane == k) y = yk;
      if (lane > k) y = fma(-row[k], yk, y);
    }
  }
  // back L^T u = y: lane l < k needs L[k][l], lane k's row[l]: the rows of L
  // are published to shared memory once
#pragma unroll
  for (int c = 0; c < 32; ++c)
    if (lane < d && c < lane) H[lane * 33 + c] = row[c];
  __syncwarp();
  double u = y;
  for (int k = d - 1; k >= 0; --k) {
    const double uk = __shfl_sync(0xffffffffu, u * rdl, k);
    if (lane == k) u = uk;
    if (lane < k) u = fma(-H[k * 33 + lane], uk, u);
  }
  if (lane < d) {
    const double xn = xs[lane] + u;
    x_next[lane] = xn;
    xs[lane] = xn;  // x^{t+1}: the next iteration's start
  }
  }  // pivots ok
  }  // warp 0
  __syncthreads();
  }  // t
}
}  // namespace

size_t small_step_smem(int64_t n, int64_t d, int64_t m, int s) {
  return small_layout((int)n, (int)d, (int)(m / s), s).total;
}

bool small_step_supported(int64_t n, int64_t d, int64_t m, int s) {
  return n >= 1 && n <= 32768 && d >= 1 && d <= 32 && s >= 1 && s <= 32 && m % s == 0 && m / s >= 1 &&
         m / s <= 32768 && (int64_t)s * n <= 65535 && small_step_smem(n, d, m, s) <= 225 * 1024;
}

cudaError_t launch_small_step(const double *A, int64_t n, int64_t d, const double *b, const double *x, uint64_t seed,
                              uint64_t iter0, int T, int64_t row_offset, int64_t m, int s, double scale, double *xout,
                              double *SA_out, double *g_out, double *H_out, int *status, cudaStream_t st,
                              LaunchCounter lc) {
  if (T < 1) return cudaSuccess;
  const size_t smem = small_step_smem(n, d, m, s);
  IHS_SMEM_ATTR(small_step_kernel, smem);
  small_step_kernel<<<1, kThreads, smem, st>>>(A, (int)n, (int)d, b, x, seed, iter0, T, row_offset, s, (int)(m / s),
                                               scale, xout, SA_out, g_out, H_out, status);
  lc.add();
  return cudaGetLastError();
}

}  // namespace ihs
