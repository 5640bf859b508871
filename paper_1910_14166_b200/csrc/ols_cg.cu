// a6, OLS for d > 160 (BASELINE.json configs[2]: d = 1024): the update
// x^{t+1} = x^t + u with H u = g (Eq. (2) with C = R^d) solved
// to machine precision by Jacobi-preconditioned conjugate gradients on the
// fp64 Gram H = (SA)^T SA.
//
// Why not the blocked Cholesky (chol_large.cu, kept behind IHS_OLS=chol): its
// critical path is d sequential pivot steps (~150-330 clocks each with B200's
// fp64 latencies: DFMA 23, rsqrt 65, shuffle 27) plus a sequential back
// substitution, ~1.2 ms at d = 1024.  H is a sketched Gram with m >= 8 d, so
// its condition number is small (~(1 + sqrt(d/m))^2 / (1 - sqrt(d/m))^2 ~ 4.4
// for C3) and CG reaches a relative residual of 1e-15 in a few tens of steps;
// the result agrees with the Cholesky solve up to rounding (reading R22).
//
// One cooperative launch: CTA k holds rows [k R, (k+1) R) of H in shared
// memory; per step it computes its slice of q = H p, publishes it, and after
// ONE grid barrier every CTA reads the whole q and performs the identical
// full-length vector updates (fixed-order reductions), so all CTAs (and all
// ranks of a replicated solve) hold bitwise-identical iterates.  p . H p <= 0
// reports IHS_ERR_NOT_SPD (reading R13) and leaves x unchanged.
#include "common.cuh"
#include "kernels.h"

namespace ihs {

namespace {
constexpr int kCgThreads = 256;
constexpr int kCgWarps = kCgThreads / 32;
constexpr int kCgMaxPer = 8;  // vector elements per thread (d <= 2048)

// Sense-free generation barrier over all CTAs of a cooperative launch.
__device__ __forceinline__ void grid_barrier(unsigned *count, volatile unsigned *gen, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g0 = *gen;
    __threadfence();
    if (atomicAdd(count, 1u) == nblocks - 1) {
      atomicExch(count, 0u);
      __threadfence();
      atomicExch((unsigned *)gen, g0 + 1);
    } else {
      while (*gen == g0) __nanosleep(20);
    }
    __threadfence();
  }
  __syncthreads();
}

// CTA-wide sums of two values in a fixed order (every thread gets both).
__device__ __forceinline__ void cta_sum2(double &a, double &b, double *red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  a = warp_sum(a);
  b = warp_sum(b);
  __syncthreads();
  if (lane == 0) {
    red[warp] = a;
    red[kCgWarps + warp] = b;
  }
  __syncthreads();
  double sa = 0.0, sb = 0.0;
#pragma unroll
  for (int w = 0; w < kCgWarps; ++w) {
    sa += red[w];
    sb += red[kCgWarps + w];
  }
  a = sa;
  b = sb;
}

__global__ void __launch_bounds__(kCgThreads) ols_cg_kernel(const double *__restrict__ H, const double *__restrict__ g,
                                                            int d, const double *__restrict__ x, double *x_next,
                                                            double *qbuf /* 2 x d */, unsigned *bar, int rows_per,
                                                            int max_iter, double tol2, int smem_rows, int *status) {
  extern __shared__ double sm[];
  double *ps = sm;                 // d: the full p, for the local rows' products
  double *Hs = sm + d;             // rows_per x d when smem_rows
  __shared__ double red[2 * kCgWarps];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int i0 = blockIdx.x * rows_per, i1 = min(d, i0 + rows_per);
  if (smem_rows)
    load_rows(Hs, H + (int64_t)i0 * d, (int64_t)(i1 - i0) * d, tid, kCgThreads);
  // full-length vectors, element c = tid + kCgThreads * k, in registers
  double u[kCgMaxPer], r[kCgMaxPer], z[kCgMaxPer], p[kCgMaxPer], dinv[kCgMaxPer];
  double rz = 0.0, gg = 0.0;
#pragma unroll
  for (int k = 0; k < kCgMaxPer; ++k) {
    const int c = tid + kCgThreads * k;
    const bool on = c < d;
    const double hd = on ? H[(int64_t)c * d + c] : 1.0;
    dinv[k] = 1.0 / hd;
    u[k] = 0.0;
    r[k] = on ? g[c] : 0.0;
    z[k] = r[k] * dinv[k];
    p[k] = z[k];
    rz += r[k] * z[k];
    gg += r[k] * r[k];
  }
  cta_sum2(rz, gg, red);
  double nonpos = 0.0, unused = 0.0;  // a non-positive diagonal entry: H is not SPD
#pragma unroll
  for (int k = 0; k < kCgMaxPer; ++k) nonpos += (dinv[k] > 0.0) ? 0.0 : 1.0;
  cta_sum2(nonpos, unused, red);
  int it = 0;
  bool not_spd = nonpos > 0.0;
  for (;;) {
    if (not_spd || !(gg > 0.0) || it >= max_iter) break;
    // p -> shared memory; q slice = H_rows p
#pragma unroll
    for (int k = 0; k < kCgMaxPer; ++k) {
      const int c = tid + kCgThreads * k;
      if (c < d) ps[c] = p[k];
    }
    __syncthreads();
    double *q = qbuf + (size_t)(it & 1) * d;
    for (int i = i0 + warp; i < i1; i += kCgWarps) {
      const double *row = smem_rows ? Hs + (size_t)(i - i0) * d : H + (int64_t)i * d;
      double t0 = 0.0, t1 = 0.0;
      int c = lane;
      for (; c + 32 < d; c += 64) {
        t0 = fma(row[c], ps[c], t0);
        t1 = fma(row[c + 32], ps[c + 32], t1);
      }
      if (c < d) t0 = fma(row[c], ps[c], t0);
      const double s = warp_sum(t0 + t1);
      if (lane == 0) q[i] = s;
    }
    grid_barrier(bar, bar + 1, gridDim.x);
    // identical full-length updates in every CTA
    double qv[kCgMaxPer];
    double pq = 0.0, dummy = 0.0;
#pragma unroll
    for (int k = 0; k < kCgMaxPer; ++k) {
      const int c = tid + kCgThreads * k;
      qv[k] = c < d ? __ldcg(q + c) : 0.0;
      pq += p[k] * qv[k];
    }
    cta_sum2(pq, dummy, red);
    if (!(pq > 0.0)) {
      not_spd = true;
      break;
    }
    const double alpha = rz / pq;
    double rz_new = 0.0, rr = 0.0;
#pragma unroll
    for (int k = 0; k < kCgMaxPer; ++k) {
      u[k] = fma(alpha, p[k], u[k]);
      r[k] = fma(-alpha, qv[k], r[k]);
      z[k] = r[k] * dinv[k];
      rz_new += r[k] * z[k];
      rr += r[k] * r[k];
    }
    cta_sum2(rz_new, rr, red);
    ++it;
    if (rr <= tol2 * gg) break;
    const double beta = rz_new / rz;
    rz = rz_new;
#pragma unroll
    for (int k = 0; k < kCgMaxPer; ++k) p[k] = fma(beta, p[k], z[k]);
    __syncthreads();  // ps is rewritten at the top of the next step
  }
  // rows of x_next are written by the CTA that owns them in the partition of
  // the vector (every CTA holds the same u)
  if (blockIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < kCgMaxPer; ++k) {
      const int c = tid + kCgThreads * k;
      if (c < d) x_next[c] = not_spd ? x[c] : x[c] + u[k];
    }
    if (tid == 0) {
      if (not_spd) set_status(status, 3 /* IHS_ERR_NOT_SPD */);
      else if (gg > 0.0 && it >= max_iter) set_status(status, 4 /* IHS_ERR_NOT_CONVERGED */);
    }
  }
}
}  // namespace

bool ols_cg_supported(int64_t d) { return d >= 1 && d <= (int64_t)kCgThreads * kCgMaxPer; }

size_t ols_cg_scratch_bytes(int64_t d) { return (size_t)2 * d * 8 + 64; }

cudaError_t launch_ols_cg(const double *H, const double *g, int64_t d, const double *x, double *x_next,
                          double *scratch, int *status, int num_sms, cudaStream_t st, LaunchCounter lc) {
  static size_t occ_smem = 0;  // occupancy cached per dynamic smem size
  static int max_per_sm = 0;
  const int rows_per = (int)((d + num_sms - 1) / num_sms);
  const int nblk = (int)((d + rows_per - 1) / rows_per);
  size_t smem = (size_t)d * 8;
  int smem_rows = 0;
  if (smem + (size_t)rows_per * d * 8 <= 160 * 1024) {
    smem += (size_t)rows_per * d * 8;
    smem_rows = 1;
  }
  IHS_SMEM_ATTR(ols_cg_kernel, smem);
  if (occ_smem != smem) {
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, ols_cg_kernel, kCgThreads, smem);
    max_per_sm = nb;
    occ_smem = smem;
  }
  if (max_per_sm * num_sms < nblk) return cudaErrorCooperativeLaunchTooLarge;
  double *qbuf = scratch;
  unsigned *bar = reinterpret_cast<unsigned *>(scratch + 2 * d);
  cudaError_t e = cudaMemsetAsync(bar, 0, 2 * sizeof(unsigned), st);
  if (e != cudaSuccess) return e;
  int di = (int)d, mi = (int)std::min<int64_t>(2000, 4 * d), sr = smem_rows;
  double tol2 = 1e-30;  // relative residual 1e-15
  void *args[] = {(void *)&H, (void *)&g, (void *)&di, (void *)&x, (void *)&x_next, (void *)&qbuf, (void *)&bar,
                  (void *)&rows_per, (void *)&mi, (void *)&tol2, (void *)&sr, (void *)&status};
  e = cudaLaunchCooperativeKernel((const void *)ols_cg_kernel, dim3(nblk), dim3(kCgThreads), args, smem, st);
  lc.add();
  return e;
}

}  // namespace ihs
