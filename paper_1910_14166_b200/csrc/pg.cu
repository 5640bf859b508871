// a6, l1 ball C = {||x||_1 <= tau} (section 1): the Eq. (2)
// quadratic program 1/2 (y-x)^T H (y-x) - g^T (y-x) over C, "solved exactly"
// by projected gradient (reading R10): step 1/L with
// L = safety * lambda_max(H) from power iteration, Euclidean projection onto
// the ball, stop when ||y+ - y|| <= tol * max(1, ||y||).  One persistent CTA
// runs every inner step (the loop is latency-bound: ~10^2 dependent steps per
// outer iteration); H stays L2-resident.  The projection threshold is found by
// Michelot's fixed-point iteration, which reaches the same theta as the sorted
// rule of the oracle (R8) in exact arithmetic.
#include "common.cuh"
#include "kernels.h"

namespace ihs {

namespace {
constexpr int kThreads = 1024;
constexpr int kWarps = kThreads / 32;

// Sum two values over the CTA; every thread gets both totals.
__device__ __forceinline__ void block_sum2(double &a, double &b, double *red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  a = warp_sum(a);
  b = warp_sum(b);
  __syncthreads();  // red may still be read from the previous call
  if (lane == 0) {
    red[warp] = a;
    red[kWarps + warp] = b;
  }
  __syncthreads();
  double sa = 0.0, sb = 0.0;
#pragma unroll 8
  for (int w = 0; w < kWarps; ++w) {
    sa += red[w];
    sb += red[kWarps + w];
  }
  a = sa;
  b = sb;
}

__global__ void __launch_bounds__(kThreads) pg_l1ball_kernel(const double *__restrict__ H,
                                                             const double *__restrict__ g, int d,
                                                             const double *__restrict__ x, double radius,
                                                             int max_inner, int power_iters, double tol,
                                                             double safety, double *x_next, int32_t *inner_iters,
                                                             int *status) {
  extern __shared__ double sm[];
  double *xs = sm;          // x^t
  double *gs = xs + d;      // g
  double *y = gs + d;       // current iterate
  double *z = y + d;        // gradient step / power-iteration vector
  double *w = z + d;        // y - x, or H v
  __shared__ double red[2 * kWarps];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < d; i += kThreads) {
    xs[i] = x[i];
    gs[i] = g[i];
    y[i] = x[i];
    z[i] = 1.0 / sqrt((double)d);
  }
  __syncthreads();
  // lambda_max(H) by power iteration from 1/sqrt(d)
  double lam = 0.0;
  for (int it = 0; it < power_iters; ++it) {
    for (int p = warp; p < d; p += kWarps) {
      const double *hr = H + (int64_t)p * d;
      double acc = 0.0;
      for (int q = lane; q < d; q += 32) acc = fma(hr[q], z[q], acc);
      acc = warp_sum(acc);
      if (lane == 0) w[p] = acc;
    }
    __syncthreads();
    double nn = 0.0, dummy = 0.0;
    for (int i = tid; i < d; i += kThreads) nn = fma(w[i], w[i], nn);
    block_sum2(nn, dummy, red);
    lam = sqrt(nn);
    if (!(lam > 0.0)) break;
    for (int i = tid; i < d; i += kThreads) z[i] = w[i] / lam;
    __syncthreads();
  }
  const double L = (lam > 0.0) ? safety * lam : 1.0;
  int k = 0;
  bool converged = false;
  while (k < max_inner) {
    for (int i = tid; i < d; i += kThreads) w[i] = y[i] - xs[i];
    __syncthreads();
    // z = y - (H (y - x) - g) / L
    for (int p = warp; p < d; p += kWarps) {
      const double *hr = H + (int64_t)p * d;
      double acc = 0.0;
      for (int q = lane; q < d; q += 32) acc = fma(hr[q], w[q], acc);
      acc = warp_sum(acc);
      if (lane == 0) z[p] = y[p] - (acc - gs[p]) / L;
    }
    __syncthreads();
    // projection onto {||.||_1 <= radius}: theta by Michelot's iteration
    double n1 = 0.0, cntd = 0.0;
    for (int i = tid; i < d; i += kThreads) n1 += fabs(z[i]);
    block_sum2(n1, cntd, red);
    double theta = 0.0;
    if (n1 > radius) {
      theta = (n1 - radius) / (double)d;
      double cprev = (double)d;
      for (int guard = 0; guard <= d; ++guard) {
        double S = 0.0, c = 0.0;
        for (int i = tid; i < d; i += kThreads) {
          double a = fabs(z[i]);
          if (a > theta) {
            S += a;
            c += 1.0;
          }
        }
        block_sum2(S, c, red);
        if (c == cprev || c == 0.0) break;
        theta = (S - radius) / c;
        cprev = c;
      }
    }
    double dn = 0.0, yy = 0.0;
    for (int i = tid; i < d; i += kThreads) {
      double zi = z[i];
      double yn = zi;
      if (n1 > radius) {
        double a = fabs(zi) - theta;
        yn = a > 0.0 ? (zi < 0.0 ? -a : a) : 0.0;
      }
      double e = yn - y[i];
      dn = fma(e, e, dn);
      yy = fma(y[i], y[i], yy);
      z[i] = yn;
    }
    block_sum2(dn, yy, red);
    for (int i = tid; i < d; i += kThreads) y[i] = z[i];
    ++k;
    if (sqrt(dn) <= tol * fmax(1.0, sqrt(yy))) {
      converged = true;
      break;
    }
    __syncthreads();
  }
  __syncthreads();
  for (int i = tid; i < d; i += kThreads) x_next[i] = y[i];
  if (tid == 0) {
    if (inner_iters) *inner_iters = k;
    if (!converged) set_status(status, 4 /* IHS_ERR_NOT_CONVERGED */);
  }
}
}  // namespace

size_t pg_scratch_bytes(int64_t d) { return 0; }

cudaError_t launch_l1ball_update(const double *H, const double *g, int64_t d, const double *x, double radius,
                                 int max_inner, int power_iters, double tol, double safety, double *x_next,
                                 int32_t *inner_iters, double *scratch, int *status, cudaStream_t st,
                                 LaunchCounter lc) {
  (void)scratch;
  const size_t smem = (size_t)5 * d * 8;
  if (smem > 200 * 1024) return cudaErrorInvalidValue;
  IHS_SMEM_ATTR(pg_l1ball_kernel, smem);
  pg_l1ball_kernel<<<1, kThreads, smem, st>>>(H, g, (int)d, x, radius, max_inner, power_iters, tol, safety, x_next,
                                              inner_iters, status);
  lc.add();
  return cudaGetLastError();
}

}  // namespace ihs
