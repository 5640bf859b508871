// a6, OLS for d > 160 (BASELINE.json configs[2]: d = 1024): the update
// x^{t+1} = x^t + u with H u = g (Eq. (2) with C = R^d; "solved
// exactly"), in ONE cooperative launch:
//
//  1. Jacobi-preconditioned conjugate gradients to a relative residual of
//     1e-15 (reading R22).  A sketched Gram with m >= 8 d is well conditioned
//     (kappa ~ (1 + sqrt(d/m))^2 / (1 - sqrt(d/m))^2 ~ 4.4 for C3), so CG takes
//     a few tens of steps; its critical path is one grid barrier per step.
//  2. If CG does not finish -- its step cap min(2000, 4d) (an ill-conditioned
//     H), or a direction with p.Hp <= 0 / a non-positive diagonal entry (H not
//     positive definite, or rounding on a nearly singular H) -- the same
//     launch continues with the blocked right-looking Cholesky of the
//     augmented matrix [[H, g], [g^T, *]] (64-column panels: potrf of the
//     diagonal block on CTA 0, the panel's triangular solve and the trailing
//     DMMA update spread over the CTAs, a grid barrier between phases; the
//     forward solve is row d of the factor; CTA 0 back-substitutes).  Its
//     verdict is the oracle's (reading R13): a pivot <= 0 sets IHS_ERR_NOT_SPD
//     and leaves x_next = x.  The whole grid takes the same branch: every CTA
//     holds the same CG scalars (fixed-order reductions).
//  The Cholesky alone (CG off) is the certified path (ihs_ctx_set_option
//  "ols_cg" = 0): CG certifies positive definiteness only on the Krylov space
//  it explores (R22).
//
// CTA k keeps rows [k R, (k+1) R) of H in shared memory for the CG products
// q = H p; after the grid barrier every CTA performs identical full-length
// vector updates, so CTAs and ranks hold bitwise-identical iterates.
#include "common.cuh"
#include "kernels.h"
#include "chol_blocks.cuh"

namespace ihs {

namespace {
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxPer = 8;  // vector elements per thread (d <= 2048)
constexpr int PB = 64;      // Cholesky panel width
constexpr int LDP = PB + 4;
constexpr int kTrsmRows = 128;

__device__ __forceinline__ void dmma884(double &c0, double &c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// Grid barrier over all CTAs of a cooperative launch: one ticket counter that
// only grows (zeroed by the launch's memset); a CTA's ticket t releases when
// the counter reaches the next multiple of the grid size.  One atomic round
// trip and a relaxed poll of the same word -- the generation-word version
// (read the generation, fence, atomic, last arriver resets the count and
// bumps the generation, the others sleep-poll it) measured ~4650 cycles per
// CG step (tools/probe/cg_timing.cu).  (`gen` is unused; kept for the
// scratch layout.)
__device__ __forceinline__ void grid_barrier(unsigned *count, volatile unsigned *gen, unsigned nblocks) {
  (void)gen;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned t;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(t) : "l"(count) : "memory");
    const unsigned target = (t / nblocks + 1u) * nblocks;
    for (;;) {
      unsigned v;
      asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(count) : "memory");
      if (v >= target) break;
    }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  __syncthreads();
}
// (Tickets spread over 8 counters 128 B apart, polled by 8 lanes, measured
// slower: 3600 vs 3150 cycles per CG step -- the arrivals were not the cost.)

// CTA-wide sums of two values in a fixed order (every thread gets both).
__device__ __forceinline__ void cta_sum2(double &a, double &b, double *red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  a = warp_sum(a);
  b = warp_sum(b);
  __syncthreads();
  if (lane == 0) {
    red[warp] = a;
    red[kWarps + warp] = b;
  }
  __syncthreads();
  double sa = 0.0, sb = 0.0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) {
    sa += red[w];
    sb += red[kWarps + w];
  }
  a = sa;
  b = sb;
}

struct Chol {
  double *M;      // Dp x Dp augmented matrix, lower triangle factored in place
  double *rdiag;  // Dp reciprocal pivots
  int *flag;      // 1 once a pivot <= 0 was met
  int Dp, d;
};

// ---- Cholesky phases (every CTA of the grid calls chol_grid) ---------------
__device__ void aug_fill(const double *__restrict__ H, const double *__restrict__ g, const Chol &c) {
  const int64_t total = (int64_t)c.Dp * c.Dp;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / c.Dp), col = (int)(e % c.Dp);
    double v = 0.0;
    if (col <= i) {
      if (i < c.d) v = H[(int64_t)i * c.d + col];
      else if (i == c.d) v = col < c.d ? g[col] : 1.0;
      else v = (col == i) ? 1.0 : 0.0;
    }
    c.M[e] = v;
  }
}

// Factor the diagonal 64x64 block at (kb, kb) in shared memory (one CTA).
__device__ void potrf_diag(const Chol &c, int kb, int *status, double *sm) {
  double *Ls = sm;             // PB x LDP
  double *rd = Ls + PB * LDP;  // PB
  double *colbuf = rd + PB;    // 64
  int *s_bad = reinterpret_cast<int *>(colbuf + 64);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = warp; i < PB; i += kWarps)
    for (int col = lane; col <= i; col += 32) Ls[i * LDP + col] = c.M[(int64_t)(kb + i) * c.Dp + kb + col];
  if (tid == 0) *s_bad = 0;
  __syncthreads();
  for (int k2 = 0; k2 < PB; k2 += 32) {
    if (warp == 0) {
      const bool bad = warp_chol32(Ls + k2 * LDP + k2, LDP, rd + k2, c.d - (kb + k2), colbuf);
      if (bad && lane == 0) *s_bad = 1;
    }
    __syncthreads();
    if (*s_bad) break;
    if (k2 == 0) {
      if (tid < 32) thread_trsm32(Ls + (32 + tid) * LDP, Ls, LDP, rd);  // rows 32..63 against the first block
      __syncthreads();
      for (int t = warp; t < 10; t += kWarps) {  // lower 8x8 tiles of the (32,32) block -= L21 L21^T
        int ti = 0, rem = t;
        while (rem > ti) {
          rem -= ti + 1;
          ++ti;
        }
        const int I = 32 + 8 * ti, J = 32 + 8 * rem;
        double c0 = 0.0, c1 = 0.0;
#pragma unroll
        for (int kk = 0; kk < 32; kk += 4)
          dmma884(c0, c1, Ls[(I + (lane >> 2)) * LDP + kk + (lane & 3)], Ls[(J + (lane >> 2)) * LDP + kk + (lane & 3)]);
        const int r = I + (lane >> 2), col = J + 2 * (lane & 3);
        Ls[r * LDP + col] -= c0;
        Ls[r * LDP + col + 1] -= c1;
      }
      __syncthreads();
    }
  }
  if (*s_bad) {
    if (tid == 0) {
      *c.flag = 1;
      set_status(status, 3 /* IHS_ERR_NOT_SPD */);
    }
    return;
  }
  for (int i = warp; i < PB; i += kWarps)
    for (int col = lane; col <= i; col += 32) c.M[(int64_t)(kb + i) * c.Dp + kb + col] = Ls[i * LDP + col];
  if (tid < PB) c.rdiag[kb + tid] = rd[tid];
}

// Rows [r0, r0 + 128) below the panel: X L11^T = A21, one thread per row
// (threads 0..127); with L11 = [[P, 0], [Q, R]]: x1 P^T = a1, x2 R^T = a2 - x1 Q^T.
__device__ void trsm_rows(const Chol &c, int kb, int r0, double *sm) {
  double *L11 = sm;                      // PB x (PB + 1)
  double *X = L11 + PB * (PB + 1);       // kTrsmRows x (PB + 1)
  double *rd = X + kTrsmRows * (PB + 1);  // PB
  for (int e = threadIdx.x; e < PB * PB; e += blockDim.x) {
    const int i = e / PB, col = e % PB;
    L11[i * (PB + 1) + col] = (col <= i) ? c.M[(int64_t)(kb + i) * c.Dp + kb + col] : 0.0;
  }
  if (threadIdx.x < PB) rd[threadIdx.x] = c.rdiag[kb + threadIdx.x];
  const int nr = min(kTrsmRows, c.Dp - r0);
  for (int e = threadIdx.x; e < nr * PB; e += blockDim.x) {
    const int r = e / PB, col = e % PB;
    X[r * (PB + 1) + col] = c.M[(int64_t)(r0 + r) * c.Dp + kb + col];
  }
  __syncthreads();
  if (threadIdx.x < nr) {
    double *x = X + threadIdx.x * (PB + 1);
    thread_trsm32(x, L11, PB + 1, rd);
    const double *Q = L11 + 32 * (PB + 1);
#pragma unroll 1
    for (int col = 0; col < 32; ++col) {
      double t0 = 0.0, t1 = 0.0;
#pragma unroll
      for (int k = 0; k < 32; k += 2) {
        t0 = fma(x[k], Q[col * (PB + 1) + k], t0);
        t1 = fma(x[k + 1], Q[col * (PB + 1) + k + 1], t1);
      }
      x[32 + col] -= t0 + t1;
    }
    thread_trsm32(x + 32, L11 + 32 * (PB + 1) + 32, PB + 1, rd + 32);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nr * PB; e += blockDim.x) {
    const int r = e / PB, col = e % PB;
    c.M[(int64_t)(r0 + r) * c.Dp + kb + col] = X[r * (PB + 1) + col];
  }
  __syncthreads();
}

// Trailing lower tile `tile` (row-major over the lower triangle below the
// panel) -= P_I P_J^T, by one 4-warp group (DMMA, 32x32 sub-tiles per warp).
__device__ void syrk_tile(const Chol &c, int kb, int tile, int wg, double *sm) {
  double *PI = sm;             // [k][r], PB x LDP
  double *PJ = sm + PB * LDP;  // [k][r]
  const int t0 = kb + PB;
  int ti = 0, rem = tile;
  while (rem > ti) {
    rem -= ti + 1;
    ++ti;
  }
  const int I = t0 + PB * ti, J = t0 + PB * rem;
  const int tid = threadIdx.x & 127, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < PB * PB; e += 128) {
    const int r = e / PB, k = e % PB;
    PI[k * LDP + r] = c.M[(int64_t)(I + r) * c.Dp + kb + k];
    PJ[k * LDP + r] = c.M[(int64_t)(J + r) * c.Dp + kb + k];
  }
  asm volatile("bar.sync %0, 128;" ::"r"(1 + wg) : "memory");
  const int wm = warp >> 1, wn = warp & 1;
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
#pragma unroll 4
  for (int kk = 0; kk < PB; kk += 4) {
    const int kr = kk + (lane & 3);
    double av[4], bv[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) av[a] = PI[kr * LDP + 32 * wm + 8 * a + (lane >> 2)];
#pragma unroll
    for (int b = 0; b < 4; ++b) bv[b] = PJ[kr * LDP + 32 * wn + 8 * b + (lane >> 2)];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) dmma884(acc[a][b][0], acc[a][b][1], av[a], bv[b]);
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int r = I + 32 * wm + 8 * a + (lane >> 2);
      const int col = J + 32 * wn + 8 * b + 2 * (lane & 3);
      double *p = c.M + (int64_t)r * c.Dp + col;
      p[0] -= acc[a][b][0];
      p[1] -= acc[a][b][1];
    }
  asm volatile("bar.sync %0, 128;" ::"r"(1 + wg) : "memory");
}

// Back substitution L^T u = y (y = row d of the augmented factor), then
// x_next = x + u; x_next = x when a pivot failed (one CTA).
__device__ void backsolve(const Chol &c, const double *__restrict__ x, double *x_next, double *sm) {
  double *z = sm;         // d
  double *Lp = sm + c.d;  // PB x (PB + 1)
  const int tid = threadIdx.x, lane = tid & 31;
  const int d = c.d;
  if (*c.flag) {
    for (int k = tid; k < d; k += blockDim.x) x_next[k] = x[k];
    return;
  }
  for (int k = tid; k < d; k += blockDim.x) z[k] = c.M[(int64_t)d * c.Dp + k];
  __syncthreads();
  for (int kb = ((d - 1) / PB) * PB; kb >= 0; kb -= PB) {
    const int w = min(PB, d - kb);
    for (int e = tid; e < PB * PB; e += blockDim.x) {
      const int i = e / PB, col = e % PB;
      Lp[i * (PB + 1) + col] = (i < w && col <= i) ? c.M[(int64_t)(kb + i) * c.Dp + kb + col] : 0.0;
    }
    __syncthreads();
    if (tid < 32) {
      double zr[2];
      zr[0] = lane < w ? z[kb + lane] : 0.0;
      zr[1] = lane + 32 < w ? z[kb + lane + 32] : 0.0;
#pragma unroll
      for (int s = 1; s >= 0; --s) {
        for (int jj = 31; jj >= 0; --jj) {
          const int i = 32 * s + jj;
          if (i >= w) continue;
          const double ui = __shfl_sync(0xffffffffu, zr[s], jj) * c.rdiag[kb + i];
          if (lane == jj) zr[s] = ui;
#pragma unroll
          for (int q = 0; q <= s; ++q) {
            const int k = lane + 32 * q;
            if (k < i) zr[q] -= Lp[i * (PB + 1) + k] * ui;
          }
        }
      }
      if (lane < w) z[kb + lane] = zr[0];
      if (lane + 32 < w) z[kb + lane + 32] = zr[1];
    }
    __syncthreads();
    // z[k] -= sum_i L[kb+i][k] u[kb+i] for k < kb (16 independent loads in flight)
    for (int k = tid; k < kb; k += blockDim.x) {
      const double *col = c.M + (int64_t)kb * c.Dp + k;
      double t0 = 0.0, t1 = 0.0;
      if (w == PB) {
#pragma unroll 16
        for (int i = 0; i < PB; i += 2) {
          t0 = fma(col[(int64_t)i * c.Dp], z[kb + i], t0);
          t1 = fma(col[(int64_t)(i + 1) * c.Dp], z[kb + i + 1], t1);
        }
      } else {
        for (int i = 0; i < w; ++i) t0 = fma(col[(int64_t)i * c.Dp], z[kb + i], t0);
      }
      z[k] -= t0 + t1;
    }
    __syncthreads();
  }
  for (int k = tid; k < d; k += blockDim.x) x_next[k] = x[k] + z[k];
}

// The blocked Cholesky solve over the whole cooperative grid.
__device__ void chol_grid(const double *H, const double *g, const double *x, double *x_next, const Chol &c,
                          int *status, unsigned *bar, double *sm) {
  if (blockIdx.x == 0 && threadIdx.x == 0) *c.flag = 0;
  aug_fill(H, g, c);
  grid_barrier(bar, bar + 1, gridDim.x);
  for (int kb = 0; kb < c.Dp; kb += PB) {
    if (blockIdx.x == 0) potrf_diag(c, kb, status, sm);
    grid_barrier(bar, bar + 1, gridDim.x);
    if (*(volatile int *)c.flag) break;  // uniform: read after the barrier
    const int below = c.Dp - kb - PB;
    if (below <= 0) break;
    for (int rb = blockIdx.x; rb * kTrsmRows < below; rb += gridDim.x) trsm_rows(c, kb, kb + PB + rb * kTrsmRows, sm);
    grid_barrier(bar, bar + 1, gridDim.x);
    const int nt = below / PB, ntiles = nt * (nt + 1) / 2;
    const int wg = threadIdx.x >> 7;  // two 4-warp groups, a tile each
    for (int t = 2 * blockIdx.x + wg; t - wg < ntiles; t += 2 * gridDim.x)
      if (t < ntiles) syrk_tile(c, kb, t, wg, sm + wg * 2 * PB * LDP);
    grid_barrier(bar, bar + 1, gridDim.x);
  }
  if (blockIdx.x == 0) backsolve(c, x, x_next, sm);
}

#ifdef IHS_CG_TIMING
// tools/probe/cg_timing.cu only (never in the library build): per-phase clock
// sums of the CG loop, measured by thread 0 of CTA 0.
__device__ long long g_cg_timing[8];
#define CGT_MARK(v) long long v = clock64()
#define CGT_ADD(i, a, b) cgt_acc[i] += (b) - (a)
#else
#define CGT_MARK(v)
#define CGT_ADD(i, a, b)
#endif

// RP > 0 (d <= 1024, at most RP rows a CTA): the CTA's rows of H in
// registers, thread t holding columns t + 256 k (k < 4) of each -- the product
// H p is then RP register dot products and one CTA reduction, with no shared-
// memory pass over H or p (1670 cycles per step with the rows in shared memory).
// RP = 0: rows in shared memory (or global), one warp per row.
template <int RP>
__global__ void __launch_bounds__(kThreads) ols_large_kernel(const double *__restrict__ H,
                                                             const double *__restrict__ g, int d,
                                                             const double *__restrict__ x, double *x_next,
                                                             double *qbuf /* 2 x d */, unsigned *bar, int rows_per,
                                                             int max_iter, double tol2, int smem_rows, int mode,
                                                             Chol chol, int *status) {
  extern __shared__ double sm[];
  __shared__ double red[2 * kWarps];
  __shared__ double redq[kWarps * (RP > 0 ? RP : 1)];
  if (mode == 2) {  // Cholesky only
    chol_grid(H, g, x, x_next, chol, status, bar, sm);
    return;
  }
  double *ps = sm;       // d: the full p, for the local rows' products
  double *Hs = sm + d;   // rows_per x d when smem_rows
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int i0 = blockIdx.x * rows_per, i1 = min(d, i0 + rows_per);
  constexpr int KR = 4;  // (RP > 0: d <= 4 * kThreads)
  double hreg[RP > 0 ? RP : 1][KR];
  if (RP > 0) {
#pragma unroll
    for (int i = 0; i < (RP > 0 ? RP : 1); ++i)
#pragma unroll
      for (int k = 0; k < KR; ++k) {
        const int c = tid + kThreads * k;
        hreg[i][k] = (i0 + i < i1 && c < d) ? __ldg(H + (int64_t)(i0 + i) * d + c) : 0.0;
      }
  } else if (smem_rows) {
    load_rows(Hs, H + (int64_t)i0 * d, (int64_t)(i1 - i0) * d, tid, kThreads);
  }
  // full-length vectors, element c = tid + kThreads * k, in registers
  double u[kMaxPer], r[kMaxPer], z[kMaxPer], p[kMaxPer], dinv[kMaxPer];
  double rz = 0.0, gg = 0.0;
#pragma unroll
  for (int k = 0; k < kMaxPer; ++k) {
    const int c = tid + kThreads * k;
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
  for (int k = 0; k < kMaxPer; ++k) nonpos += (dinv[k] > 0.0) ? 0.0 : 1.0;
  cta_sum2(nonpos, unused, red);
  int it = 0;
  bool not_spd = nonpos > 0.0;
#ifdef IHS_CG_TIMING
  long long cgt_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#endif
  for (;;) {
    if (not_spd || !(gg > 0.0) || it >= max_iter) break;
    CGT_MARK(c0);
    double *q = qbuf + (size_t)(it & 1) * d;
    if (RP > 0) {
      double part[RP > 0 ? RP : 1];
#pragma unroll
      for (int i = 0; i < (RP > 0 ? RP : 1); ++i) {
        double a = 0.0;
#pragma unroll
        for (int k = 0; k < KR; ++k) a = fma(hreg[i][k], p[k], a);
        part[i] = a;
      }
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1)
#pragma unroll
        for (int i = 0; i < (RP > 0 ? RP : 1); ++i) part[i] += __shfl_xor_sync(0xffffffffu, part[i], o);
      if (lane == 0)
#pragma unroll
        for (int i = 0; i < (RP > 0 ? RP : 1); ++i) redq[warp * (RP > 0 ? RP : 1) + i] = part[i];
      __syncthreads();
      if (tid < (RP > 0 ? RP : 1) && i0 + tid < i1) {
        double sq = 0.0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) sq += redq[w * (RP > 0 ? RP : 1) + tid];
        q[i0 + tid] = sq;
      }
    } else {
#pragma unroll
      for (int k = 0; k < kMaxPer; ++k) {
        const int c = tid + kThreads * k;
        if (c < d) ps[c] = p[k];
      }
      __syncthreads();
      for (int i = i0 + warp; i < i1; i += kWarps) {
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
    }
    CGT_MARK(c1);
    grid_barrier(bar, bar + 1, gridDim.x);
    CGT_MARK(c2);
    double qv[kMaxPer];
    double pq = 0.0, dummy = 0.0;
#pragma unroll
    for (int k = 0; k < kMaxPer; ++k) {
      const int c = tid + kThreads * k;
      qv[k] = c < d ? __ldcg(q + c) : 0.0;
      pq += p[k] * qv[k];
    }
    cta_sum2(pq, dummy, red);
    CGT_MARK(c3);
    if (!(pq > 0.0)) {
      not_spd = true;
      break;
    }
    const double alpha = rz / pq;
    double rz_new = 0.0, rr = 0.0;
#pragma unroll
    for (int k = 0; k < kMaxPer; ++k) {
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
    for (int k = 0; k < kMaxPer; ++k) p[k] = fma(beta, p[k], z[k]);
    __syncthreads();  // ps is rewritten at the top of the next step
    CGT_MARK(c4);
    CGT_ADD(0, c0, c1);
    CGT_ADD(1, c1, c2);
    CGT_ADD(2, c2, c3);
    CGT_ADD(3, c3, c4);
    CGT_ADD(4, c0, c4);
  }
#ifdef IHS_CG_TIMING
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    for (int i = 0; i < 5; ++i) g_cg_timing[i] = cgt_acc[i];
    g_cg_timing[5] = it;
  }
#endif
  const bool capped = gg > 0.0 && it >= max_iter && !not_spd;
  if (mode == 1 && (not_spd || capped)) {  // CG did not finish: the Cholesky decides (same launch)
    grid_barrier(bar, bar + 1, gridDim.x);  // every CTA is done with H's rows in shared memory
    chol_grid(H, g, x, x_next, chol, status, bar, sm);
    return;
  }
  if (blockIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < kMaxPer; ++k) {
      const int c = tid + kThreads * k;
      if (c < d) x_next[c] = not_spd ? x[c] : x[c] + u[k];
    }
    if (tid == 0) {
      if (not_spd) set_status(status, 3 /* IHS_ERR_NOT_SPD */);
      else if (capped) set_status(status, 4 /* IHS_ERR_NOT_CONVERGED */);
    }
  }
}

size_t chol_smem() {
  const size_t potrf = ((size_t)PB * LDP + PB + 64) * 8 + 16;
  const size_t trsm = ((size_t)(PB + kTrsmRows) * (PB + 1) + PB) * 8;
  const size_t syrk = (size_t)2 * 2 * PB * LDP * 8;
  return std::max(potrf, std::max(trsm, syrk));
}
}  // namespace

bool ols_large_supported(int64_t d) { return d >= 1 && d <= (int64_t)kThreads * kMaxPer; }

constexpr int kFlagDoubles = 8;  // the grid-barrier words
size_t ols_large_scratch_bytes(int64_t d) {
  const int64_t Dp = (d + 1 + PB - 1) / PB * PB;
  return (size_t)2 * d * 8 + kFlagDoubles * 8 + (size_t)(Dp * Dp + Dp) * 8 + 64;
}

cudaError_t launch_ols_large(const double *H, const double *g, int64_t d, const double *x, double *x_next,
                             double *scratch, int *status, int num_sms, int mode, cudaStream_t st,
                             LaunchCounter lc) {
  static size_t occ_smem = 0;  // occupancy cached per dynamic smem size
  static int max_per_sm = 0;
  const int rows_per = (int)((d + num_sms - 1) / num_sms);
  const int nblk = (int)((d + rows_per - 1) / rows_per);
  size_t smem = (size_t)d * 8;
  int smem_rows = 0;
  if (mode != 2 && smem + (size_t)rows_per * d * 8 <= 160 * 1024) {
    smem += (size_t)rows_per * d * 8;
    smem_rows = 1;
  }
  smem = std::max(smem, chol_smem());
  smem = std::max(smem, ((size_t)d + PB * (PB + 1)) * 8);  // back substitution
  // the register-row kernel when d <= 1024 and at most 8 rows a CTA
  const int rp = (mode != 2 && d <= 4 * kThreads && rows_per <= 8) ? rows_per : 0;
  const void *kern = nullptr;
  switch (rp) {
    case 1: kern = (const void *)ols_large_kernel<1>; break;
    case 2: kern = (const void *)ols_large_kernel<2>; break;
    case 3: kern = (const void *)ols_large_kernel<3>; break;
    case 4: kern = (const void *)ols_large_kernel<4>; break;
    case 5: kern = (const void *)ols_large_kernel<5>; break;
    case 6: kern = (const void *)ols_large_kernel<6>; break;
    case 7: kern = (const void *)ols_large_kernel<7>; break;
    case 8: kern = (const void *)ols_large_kernel<8>; break;
    default: kern = (const void *)ols_large_kernel<0>;
  }
  if (rp > 0) smem_rows = 0;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  static const void *occ_kern = nullptr;
  if (occ_smem != smem || occ_kern != kern) {
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, kThreads, smem);
    max_per_sm = nb;
    occ_smem = smem;
    occ_kern = kern;
  }
  if (max_per_sm * num_sms < nblk) return cudaErrorCooperativeLaunchTooLarge;
  double *qbuf = scratch;
  unsigned *bar = reinterpret_cast<unsigned *>(scratch + 2 * d);  // [2] grid-barrier words
  Chol chol;
  chol.Dp = (int)((d + 1 + PB - 1) / PB * PB);
  chol.d = (int)d;
  chol.M = scratch + 2 * d + kFlagDoubles;
  chol.rdiag = chol.M + (size_t)chol.Dp * chol.Dp;
  chol.flag = reinterpret_cast<int *>(chol.rdiag + chol.Dp);
  cudaError_t e = cudaMemsetAsync(bar, 0, 2 * sizeof(unsigned), st);
  if (e != cudaSuccess) return e;
  int di = (int)d, mi = (int)std::min<int64_t>(2000, 4 * d), sr = smem_rows, md = mode;
  double tol2 = 1e-30;  // relative residual 1e-15
  void *args[] = {(void *)&H,    (void *)&g,    (void *)&di,  (void *)&x,    (void *)&x_next,
                  (void *)&qbuf, (void *)&bar,  (void *)&rows_per, (void *)&mi, (void *)&tol2,
                  (void *)&sr,   (void *)&md,   (void *)&chol, (void *)&status};
  e = cudaLaunchCooperativeKernel(kern, dim3(nblk), dim3(kThreads), args, smem, st);
  lc.add();
  return e;
}

}  // namespace ihs
