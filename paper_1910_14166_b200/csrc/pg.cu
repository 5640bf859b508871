// a6, l1 ball C = {||x||_1 <= tau} (section 1): the Eq. (2)
// quadratic program 1/2 (y-x)^T H (y-x) - g^T (y-x) over C, "solved exactly"
// by projected gradient (reading R10): step 1/L with
// L = safety * lambda_max(H) from power iteration, Euclidean projection onto
// the ball, stop when ||y+ - y|| <= tol * max(1, ||y||).  One persistent CTA
// runs every inner step (the loop is latency-bound: ~10^2 dependent steps per
// outer iteration); H stays L2-resident.  The projection threshold is found by
// Michelot's fixed-point iteration, which reaches the same theta as the sorted
// rule of the oracle (R8) in exact arithmetic.
#include <algorithm>
#include <type_traits>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "kernels.h"

#include <cooperative_groups.h>

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

// ----------------------------------------------------------------------------
// Cluster version: CS CTAs (one thread-block cluster) keep H in distributed
// shared memory -- CTA r holds rows [r R, (r+1) R) -- so no inner step touches
// L2.  Each step: local GEMV rows -> z rows, written into every CTA's z buffer
// through DSMEM (double-buffered by step parity), one cluster barrier, then
// every CTA runs the identical projection / convergence test on the full
// vector (same inputs, same code => bitwise-identical y in all CTAs).
constexpr int kCT = 256;
constexpr int kCW = kCT / 32;

__device__ __forceinline__ void csum2(double &a, double &b, double *red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  a = warp_sum(a);
  b = warp_sum(b);
  __syncthreads();
  if (lane == 0) {
    red[warp] = a;
    red[kCW + warp] = b;
  }
  __syncthreads();
  double sa = 0.0, sb = 0.0;
#pragma unroll
  for (int w = 0; w < kCW; ++w) {
    sa += red[w];
    sb += red[kCW + w];
  }
  a = sa;
  b = sb;
}

__global__ void __launch_bounds__(kCT) pg_cluster_kernel(const double *__restrict__ H, const double *__restrict__ g,
                                                         int d, const double *__restrict__ x, double radius,
                                                         int max_inner, int power_iters, double tol, double safety,
                                                         double *x_next, int32_t *inner_iters, int *status) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int cs = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  const int R = (d + cs - 1) / cs;
  const int r0 = rank * R, r1 = min(d, r0 + R);
  extern __shared__ double sm[];
  double *Hs = sm;                   // R x d (my rows)
  double *xs = Hs + (size_t)R * d;   // d
  double *gs = xs + d;               // d
  double *y = gs + d;                // d
  double *w = y + d;                 // d : y - x, or the power-iteration vector
  double *zb = w + d;                // 2 x d : z (or H v), double-buffered by step parity
  __shared__ double red[2 * kCW];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  load_rows(Hs, H + (int64_t)r0 * d, (int64_t)(r1 - r0) * d, tid, kCT);
  for (int i = tid; i < d; i += kCT) {
    xs[i] = x[i];
    gs[i] = g[i];
    y[i] = x[i];
    w[i] = 1.0 / sqrt((double)d);
  }
  cluster.sync();
  int par = 0;
  // my rows of H v (or H (y - x)) -> every CTA's zb[par]
  auto gemv_bcast = [&](bool pg_step, double L) {
    double *dst = cluster.map_shared_rank(zb + par * d, lane < cs ? lane : 0);  // lane r writes CTA r
    for (int p = r0 + warp; p < r1; p += kCW) {
      const double *hr = Hs + (size_t)(p - r0) * d;
      double acc = 0.0;
      for (int q = lane; q < d; q += 32) acc = fma(hr[q], w[q], acc);
      acc = warp_sum(acc);
      const double val = pg_step ? y[p] - (acc - gs[p]) / L : acc;
      if (lane < cs) dst[p] = val;
    }
    cluster.sync();
  };
  double lam = 0.0;
  for (int it = 0; it < power_iters; ++it) {
    gemv_bcast(false, 1.0);
    const double *hv = zb + par * d;
    double nn = 0.0, dummy = 0.0;
    for (int i = tid; i < d; i += kCT) nn = fma(hv[i], hv[i], nn);
    csum2(nn, dummy, red);
    lam = sqrt(nn);
    if (!(lam > 0.0)) break;
    for (int i = tid; i < d; i += kCT) w[i] = hv[i] / lam;
    par ^= 1;
    __syncthreads();
  }
  const double L = (lam > 0.0) ? safety * lam : 1.0;
  int k = 0;
  bool converged = false;
  while (k < max_inner) {
    for (int i = tid; i < d; i += kCT) w[i] = y[i] - xs[i];
    __syncthreads();
    gemv_bcast(true, L);
    const double *z = zb + par * d;
    double n1 = 0.0, dummy = 0.0;
    for (int i = tid; i < d; i += kCT) n1 += fabs(z[i]);
    csum2(n1, dummy, red);
    double theta = 0.0;
    if (n1 > radius) {
      theta = (n1 - radius) / (double)d;
      double cprev = (double)d;
      for (int guard = 0; guard <= d; ++guard) {
        double S = 0.0, c = 0.0;
        for (int i = tid; i < d; i += kCT) {
          const double a = fabs(z[i]);
          if (a > theta) {
            S += a;
            c += 1.0;
          }
        }
        csum2(S, c, red);
        if (c == cprev || c == 0.0) break;
        theta = (S - radius) / c;
        cprev = c;
      }
    }
    double dn = 0.0, yy = 0.0;
    for (int i = tid; i < d; i += kCT) {
      const double zi = z[i];
      double yn = zi;
      if (n1 > radius) {
        const double a = fabs(zi) - theta;
        yn = a > 0.0 ? (zi < 0.0 ? -a : a) : 0.0;
      }
      const double e = yn - y[i];
      dn = fma(e, e, dn);
      yy = fma(y[i], y[i], yy);
      w[i] = yn;  // staged: y is still read by other threads of this CTA above
    }
    csum2(dn, yy, red);
    for (int i = tid; i < d; i += kCT) y[i] = w[i];
    par ^= 1;
    ++k;
    if (sqrt(dn) <= tol * fmax(1.0, sqrt(yy))) {
      converged = true;
      break;
    }
    __syncthreads();
  }
  cluster.sync();  // no CTA may exit while others can still write into its shared memory
  if (rank == 0) {
    for (int i = tid; i < d; i += kCT) x_next[i] = y[i];
    if (tid == 0) {
      if (inner_iters) *inner_iters = k;
      if (!converged) set_status(status, 4 /* IHS_ERR_NOT_CONVERGED */);
    }
  }
}


// ----------------------------------------------------------------------------
// Warp-redundant cluster version for d <= 32 K (K <= 8 per lane): as above, but
// every WARP holds the whole iterate in registers (element q = lane + 32 k) and
// runs the projection, the norms and the convergence test on its own with
// warp shuffles -- all warps of all CTAs compute bitwise-identical values --
// so an inner step has no CTA barrier, only the one cluster barrier after the
// z rows are exchanged.  The GEMV interleaves a warp's rows (independent fp64
// chains) and reduces them with one transpose-reduce.
#ifdef IHS_PG_TIMING
// tools/probe/pg_timing.cu only (never in the library build): per-phase clock
// sums of the inner loop, measured by thread 0 of cluster rank 0.
__device__ long long g_pg_timing[8];
#define PGT_MARK(v) long long v = clock64()
#define PGT_ADD(i, a, b) pgt_acc[i] += (b) - (a)
#else
#define PGT_MARK(v)
#define PGT_ADD(i, a, b)
#endif

// The z exchange without a cluster barrier: every owner lane sends its row
// value to each CTA with st.async, which completes bytes on the RECEIVING
// CTA's mbarrier for that buffer; a CTA waits on its own mbarrier only (d * 8
// bytes per step, armed by its thread 0).  Reuse of buffer par two steps later
// is safe: a CTA can only send step k+2 rows after its step k+1 wait, which
// needs every CTA's step k+1 rows, which each CTA sends only after it has read
// its step k z.
__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t cluster_addr(uint32_t local, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_async_f64(uint32_t addr, double v, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(addr),
               "l"(__double_as_longlong(v)), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void zbar_arm(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void zbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "ZW_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra ZW_%=;\n\t}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

// FISTA momentum (t_{j+1} = (1 + sqrt(1 + 4 t_j^2)) / 2 from t_0 = 1, coef_j =
// (t_j - 1) / t_{j+1}), tabulated at compile time for the first kFistaTab steps
// after a (re)start; later steps compute it.
constexpr int kFistaTab = 128;
constexpr double cx_sqrt(double x) {
  double r = x > 1.0 ? x : 1.0;
  for (int i = 0; i < 200; ++i) r = 0.5 * (r + x / r);
  return r;
}
struct FistaTab {
  double c[kFistaTab];
  double t_last;
  constexpr FistaTab() : c(), t_last(1.0) {
    double t = 1.0;
    for (int j = 0; j < kFistaTab; ++j) {
      const double tn = 0.5 * (1.0 + cx_sqrt(1.0 + 4.0 * t * t));
      c[j] = (t - 1.0) / tn;
      t = tn;
    }
    t_last = t;
  }
};
__constant__ FistaTab kFista = FistaTab();
__device__ __forceinline__ double fista_coef(int j) {
  if (j < kFistaTab) return kFista.c[j];
  double t = kFista.t_last;  // (rare: > 128 steps without a restart)
  double tn = t;
  for (int i = kFistaTab; i <= j; ++i) {
    tn = 0.5 * (1.0 + sqrt(1.0 + 4.0 * t * t));
    if (i < j) t = tn;
  }
  return (t - 1.0) / tn;
}

template <int K>
__device__ __forceinline__ double wsum_k(const double (&v)[K]) {
  double t = 0.0;
#pragma unroll
  for (int k = 0; k < K; ++k) t += v[k];
  return warp_sum(t);
}

// 4 warps (one per SM sub-partition: every warp repeats the projection and
// the norms on the whole iterate, and 8 warps share the fp64 pipe for that:
// measured +250 cycles per step); warp w of cluster rank c holds rows
// c R + w U .. + U - 1 of H in registers (U x K doubles per lane, U K <= 32),
// so the H v product of an inner step reads no shared memory (with H in
// shared memory a step read R d doubles through the 128 B/clk pipe: ~512
// cycles of the ~1290-cycle product at d = 256 on 8 CTAs).
constexpr int kWT = 128;
constexpr int kWW = kWT / 32;

template <int K, int U>
__global__ void __launch_bounds__(kWT, 1) pg_warp_kernel(const double *__restrict__ H, const double *__restrict__ g,
                                                      int d, const double *__restrict__ x, double radius,
                                                      int max_inner, int power_iters, double tol, double safety,
                                                      double *x_next, int32_t *inner_iters, int *status, int accel,
                                                      double *evec, int warm, int prox, const double *L_in,
                                                      double *L_out) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int cs = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  const int R = (d + cs - 1) / cs;
  const int r0 = rank * R, r1 = min(d, r0 + R);
  extern __shared__ double sm[];
  double *gs = sm;      // R (my rows of g)
  double *zb = gs + R;  // 2 x d : z (or H v), double-buffered by step parity
  uint64_t *zbar = reinterpret_cast<uint64_t *>(zb + 2 * d);  // 2 mbarriers: zb[0], zb[1] complete
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&zbar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&zbar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const int pw = r0 + U * warp;  // this warp's first row
  double hreg[U][K];
#pragma unroll
  for (int u = 0; u < U; ++u)
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int q = lane + 32 * k;
      hreg[u][k] = (pw + u < r1 && q < d) ? __ldg(H + (int64_t)(pw + u) * d + q) : 0.0;
    }
  for (int i = tid; i < r1 - r0; i += kWT) gs[i] = g ? g[r0 + i] : 0.0;
  double xv[K], yv[K], vv[K], wv[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int q = lane + 32 * k;
    xv[k] = (q < d && x) ? x[q] : 0.0;
    yv[k] = xv[k];
    vv[k] = yv[k];
    // power iteration start: 1/sqrt(d) (reading R10), or, warm, the previous
    // call's final vector (consecutive IHS Hessian sketches are close)
    wv[k] = q < d ? (warm ? evec[q] : 1.0 / sqrt((double)d)) : 0.0;
  }
  cluster.sync();
  int par = 0;
  uint32_t zph = 0;  // bit b: the phase parity of zbar[b]
#ifdef IHS_PG_TIMING
  long long pgt_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#endif
  // rows p of this warp: out_p = pg ? y_p - ((H w)_p - g_p) / L : (H w)_p,
  // sent into every CTA's zb[par]; then this CTA's wait for all d rows.
  auto gemv_bcast = [&](bool pg_step, double invL) {
    if (tid == 0) zbar_arm(&zbar[par], (uint32_t)d * 8u);
    double acc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      double a = 0.0;
#pragma unroll
      for (int k = 0; k < K; ++k) a = fma(hreg[u][k], wv[k], a);
      acc[u] = a;
    }
    transpose_reduce<U>(acc, lane);
    const int u = reduced_row_of_lane<U>(lane);
    const int p = pw + u;
    double val = acc[0];
    if (pg_step) {  // warp-uniform; the shuffles run in every lane
      // y_p is held by lane p % 32 as element p / 32 of every warp's copy
      double yp = 0.0;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const double t = __shfl_sync(0xffffffffu, vv[k], p & 31);
        if ((p >> 5) == k) yp = t;
      }
      if (p < r1) val = fma(-(val - gs[p - r0]), invL, yp);
    }
    // the row's owner lane publishes it to every CTA of the cluster
    if (owner_lane_of_row<U>(u) == lane && p < r1) {
      const uint32_t za = smem_addr(zb + par * d + p), ba = smem_addr(&zbar[par]);
      for (int r = 0; r < cs; ++r) st_async_f64(cluster_addr(za, r), val, cluster_addr(ba, r));
    }
    PGT_MARK(tw0);
    zbar_wait(&zbar[par], (zph >> par) & 1u);
    PGT_MARK(tw1);
    PGT_ADD(1, tw0, tw1);
    zph ^= 1u << par;
  };
  // L_in: the step bound was formed beside the previous pass (look-ahead,
  // api.cu) -- no power iteration here
  double lam = 0.0;
  for (int it = 0; !L_in && it < power_iters; ++it) {
    gemv_bcast(false, 1.0);
    const double *hv = zb + par * d;
    double hvv[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int q = lane + 32 * k;
      hvv[k] = q < d ? hv[q] : 0.0;
    }
    double sq[K];
#pragma unroll
    for (int k = 0; k < K; ++k) sq[k] = hvv[k] * hvv[k];
    lam = sqrt(wsum_k(sq));
    if (!(lam > 0.0)) break;
#pragma unroll
    for (int k = 0; k < K; ++k) wv[k] = hvv[k] / lam;
    par ^= 1;
  }
  const double L = L_in ? *L_in : (lam > 0.0) ? safety * lam : 1.0;
  const double invL = 1.0 / L;
  if (!L_in && evec && rank == 0 && warp == 0 && lam > 0.0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int q = lane + 32 * k;
      if (q < d) evec[q] = wv[k];
    }
  }
  if (L_out) {  // power-only launch (the look-ahead's step bound for the next update)
    if (rank == 0 && tid == 0) *L_out = L;
    cluster.sync();
    return;
  }
  int kk = 0;
  bool converged = false;
  int tj = 0;  // FISTA: steps since the last restart (accel) -- plain PG keeps vv = yv
  double theta_prev = 0.0;  // the last projection threshold (warm start; IHS_PG_THETA_WARM=0: off)
  while (kk < max_inner) {
    PGT_MARK(ts0);
#pragma unroll
    for (int k = 0; k < K; ++k) wv[k] = vv[k] - xv[k];
    gemv_bcast(true, invL);
    PGT_MARK(ts1);
    const double *z = zb + par * d;
    double zv[K], av[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int q = lane + 32 * k;
      zv[k] = q < d ? z[q] : 0.0;
      av[k] = fabs(zv[k]);
    }
    // prox (NEXT-2, reading R23): soft threshold at lambda / L, lambda = radius;
    // else the projection onto the ball of that radius
    const double n1 = prox ? 0.0 : wsum_k(av);
    double theta = prox ? radius / L : 0.0;
    const bool proj = prox || n1 > radius;
    if (!prox && proj) {  // Michelot's fixed point (reading R19), warp-local
      // Warm start from the previous inner step's threshold: from any theta
      // above theta* one update lands at or below it (the update's active set
      // is a subset of the true one), and from below the iteration rises
      // monotonically to theta*, stopping when the active set repeats -- the
      // same final set, hence the same theta, as the cold start (n1 - tau) / d.
      bool warm_th = (accel & 2) && theta_prev > 0.0;
      theta = warm_th ? theta_prev : (n1 - radius) / (double)d;
      double cprev = warm_th ? -1.0 : (double)d;
      for (int guard = 0; guard <= d + 1; ++guard) {
        double Sh[2] = {0.0, 0.0};
        int ci = 0;  // the active count from ballots (exact; no shuffle chain)
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const bool act = av[k] > theta;
          Sh[k & 1] += act ? av[k] : 0.0;
          ci += __popc(__ballot_sync(0xffffffffu, act));
        }
        const double Sv = warp_sum(Sh[0] + Sh[1]);
        const double cv = (double)ci;
        if (cv == 0.0 && warm_th) {  // started above every |z|: cold start instead
          warm_th = false;
          theta = (n1 - radius) / (double)d;
          cprev = (double)d;
          continue;
        }
        if (cv == cprev || cv == 0.0) break;
        theta = (Sv - radius) / cv;
        cprev = cv;
      }
      theta_prev = theta;
    }
    PGT_MARK(ts2);
    // ||y+ - y||^2, ||y||^2 and the restart test in ONE interleaved warp
    // reduction; FISTA's momentum from a table (no sqrt / divide on the step's
    // critical path); convergence compared in squares.
    // y+ = sign(z) max(|z| - theta, 0) (theta = 0: y+ = z), branch-free so the
    // K elements' dependent chains interleave; each sum as two half chains.
    double ynv[K], s3[2][3] = {{0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}};
    const double th = proj ? theta : 0.0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const double yn = copysign(fmax(av[k] - th, 0.0), zv[k]);
      const double e = yn - yv[k];
      double *t3 = s3[k & 1];
      t3[0] = fma(e, e, t3[0]);
      t3[1] = fma(yv[k], yv[k], t3[1]);
      t3[2] = fma(vv[k] - yn, e, t3[2]);  // gradient-based restart test (O'Donoghue & Candes)
      ynv[k] = yn;
    }
    double s3s[3] = {s3[0][0] + s3[1][0], s3[0][1] + s3[1][1], s3[0][2] + s3[1][2]};
    PGT_MARK(tn0);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1)
#pragma unroll
      for (int i = 0; i < 3; ++i) s3s[i] += __shfl_xor_sync(0xffffffffu, s3s[i], o);
    const double dnn = s3s[0], yyy = s3s[1];
    PGT_MARK(tn1);
    PGT_ADD(5, ts2, tn0);
    PGT_ADD(6, tn0, tn1);
    if (accel & 1) {
      double coef = 0.0;
      if (s3s[2] > 0.0) {
        tj = 0;  // restart: the next step is a plain projected-gradient step
      } else {
        coef = fista_coef(tj);
        ++tj;
      }
#pragma unroll
      for (int k = 0; k < K; ++k) vv[k] = fma(coef, ynv[k] - yv[k], ynv[k]);
    } else {
#pragma unroll
      for (int k = 0; k < K; ++k) vv[k] = ynv[k];
    }
#pragma unroll
    for (int k = 0; k < K; ++k) yv[k] = ynv[k];
    par ^= 1;
    ++kk;
    PGT_MARK(ts3);
    PGT_ADD(0, ts0, ts1);
    PGT_ADD(2, ts1, ts2);
    PGT_ADD(3, ts2, ts3);
    PGT_ADD(4, ts0, ts3);
    if (dnn <= tol * tol * fmax(1.0, yyy)) {  // ||y+ - y|| <= tol max(1, ||y||)
      converged = true;
      break;
    }
  }
  cluster.sync();  // no CTA may exit while others can still write into its shared memory
#ifdef IHS_PG_TIMING
  if (rank == 0 && tid == 0)
    for (int i = 0; i < 8; ++i) g_pg_timing[i] = pgt_acc[i];
#endif
  if (rank == 0 && warp == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int q = lane + 32 * k;
      if (q < d) x_next[q] = yv[k];
    }
    if (lane == 0) {
      if (inner_iters) *inner_iters = kk;
      if (!converged) set_status(status, 4 /* IHS_ERR_NOT_CONVERGED */);
    }
  }
}

}  // namespace

int pg_cluster_size(int64_t d) {
  for (int cs : {1, 2, 4, 8, 16}) {
    const int64_t R = (d + cs - 1) / cs;
    if ((size_t)(R * d + 6 * d) * 8 <= 200 * 1024) return cs;
  }
  return 0;
}

bool lasso_supported(int64_t d) { return d >= 1 && d <= 256; }

bool pg_supported(int64_t d) { return d <= 256 || pg_cluster_size(d) > 0 || (size_t)5 * d * 8 <= 200 * 1024; }

size_t pg_scratch_bytes(int64_t d) { return (size_t)d * 8; }

cudaError_t launch_l1ball_update(const double *H, const double *g, int64_t d, const double *x, double radius,
                                 int max_inner, int power_iters, int warm_power_iters, double tol, double safety,
                                 double *x_next, int32_t *inner_iters, double *scratch, int *status, cudaStream_t st,
                                 LaunchCounter lc, bool warm_start, int prox, const double *L_in, double *L_out,
                                 int cluster_pref) {
  // d <= 256: the warp-per-iterate cluster kernel with H in registers; larger
  // d: the CTA-level cluster kernel while H fits the cluster's shared memory,
  // else one CTA.
  if (d <= 256) {
    // K doubles of the iterate per lane; U rows of H per warp (4 warps a CTA):
    // the smallest cluster with U <= 8 and U K <= 32 -- d = 256: 16 CTAs (U = 4),
    // d = 128: 4 (U = 8), d = 64: 2 (U = 8), d <= 32: 1.  cluster_pref (a power
    // of two <= 16) overrides when its U satisfies the same bounds.
    const int K = d <= 32 ? 1 : d <= 64 ? 2 : d <= 128 ? 4 : 8;
    auto u_of = [&](int c) {
      const int64_t rows = (d + c - 1) / c, per = (rows + kWW - 1) / kWW;
      return per <= 1 ? 1 : per <= 2 ? 2 : per <= 4 ? 4 : per <= 8 ? 8 : 16;
    };
    int cs = 1;
    while (cs < 16 && (u_of(cs) > 8 || u_of(cs) * K > 32)) cs *= 2;
    if (cluster_pref > 0 && cluster_pref <= 16 && (cluster_pref & (cluster_pref - 1)) == 0 &&
        u_of(cluster_pref) <= 8 && u_of(cluster_pref) * K <= 32)
      cs = cluster_pref;
    const int U = u_of(cs);
    const int64_t R = (d + cs - 1) / cs;
    const size_t smem = std::max((size_t)(R + 2 * d) * 8 + 16, kExclusiveSmem);
    const void *kern = nullptr;
#define IHS_PGK(KV, UV) \
  if (K == KV && U == UV) kern = (const void *)pg_warp_kernel<KV, UV>;
    IHS_PGK(8, 1) IHS_PGK(8, 2) IHS_PGK(8, 4) IHS_PGK(4, 1) IHS_PGK(4, 2) IHS_PGK(4, 4) IHS_PGK(4, 8)
    IHS_PGK(2, 1) IHS_PGK(2, 2) IHS_PGK(2, 4) IHS_PGK(2, 8) IHS_PGK(1, 1) IHS_PGK(1, 2) IHS_PGK(1, 4) IHS_PGK(1, 8)
#undef IHS_PGK
    if (!kern) return cudaErrorInvalidValue;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (cs > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(kWT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    lc.add();
    // accel bit 0: FISTA with restart; bit 1: warm-started projection threshold
    int accel = 3;
    // warm start (scratch = d doubles holding the last eigenvector estimate):
    // warm_power_iters steps from it instead of power_iters from 1/sqrt(d)
    const bool warm_ok = warm_start && scratch;
    int piters = warm_ok ? warm_power_iters : power_iters;
    int warm = warm_ok ? 1 : 0;
    void *args[] = {(void *)&H,     (void *)&g,         (void *)&d,        (void *)&x,      (void *)&radius,
                    (void *)&max_inner, (void *)&piters, (void *)&tol,     (void *)&safety, (void *)&x_next,
                    (void *)&inner_iters, (void *)&status, (void *)&accel, (void *)&scratch, (void *)&warm,
                    (void *)&prox,  (void *)&L_in,      (void *)&L_out};
    int di = (int)d;
    args[2] = (void *)&di;
    return cudaLaunchKernelExC(&cfg, kern, args);
  }
  int cs = pg_cluster_size(d);
  if (cs > 0) {
    if (prox || L_out) return cudaErrorNotSupported;
    const int64_t R = (d + cs - 1) / cs;
    const size_t smem = std::max((size_t)(R * d + 6 * d) * 8, kExclusiveSmem);
    cudaFuncSetAttribute((const void *)pg_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (cs > 8)
      cudaFuncSetAttribute((const void *)pg_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(kCT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    lc.add();
    return cudaLaunchKernelEx(&cfg, pg_cluster_kernel, H, g, (int)d, x, radius, max_inner, power_iters, tol, safety,
                              x_next, inner_iters, status);
  }
  if (L_out) return cudaErrorNotSupported;  // power-only launches: the warp kernel only
  if (prox) return cudaErrorNotSupported;
  const size_t smem = (size_t)5 * d * 8;
  if (smem > 200 * 1024) return cudaErrorInvalidValue;
  IHS_SMEM_ATTR(pg_l1ball_kernel, smem);
  pg_l1ball_kernel<<<1, kThreads, smem, st>>>(H, g, (int)d, x, radius, max_inner, power_iters, tol, safety, x_next,
                                              inner_iters, status);
  lc.add();
  return cudaGetLastError();
}

}  // namespace ihs
