// a6, OLS: x^{t+1} = x^t + H^{-1} g (Eq. (2) with C = R^d, PAPER.md:83-86;
// T_solve = O(d^3)).  Right-looking Cholesky H = L L^T in
// one CTA (H in shared memory when d^2 * 8 fits, else in an L2-resident global
// scratch), then forward / back substitution by one warp and the update
// x + u.  A pivot <= 0 sets IHS_ERR_NOT_SPD (reading R13) and x_next = x.
// Latency-bound: d = 10..256 take O(d) barrier steps.
#include "common.cuh"
#include "kernels.h"

#include <utility>

namespace ihs {

namespace {
constexpr int kThreads = 512;
constexpr size_t kSmemLimit = 200 * 1024;

// Right-looking elimination with ONE barrier per column: step j subtracts
// a_ij a_cj / a_jj from the trailing lower triangle (j < c <= i) while column
// j itself stays unscaled; a final pass turns the stored (a_ij, a_jj) into
// L_ij = a_ij / sqrt(a_jj).  The row stride is d + 1 so the column reads
// a_cj of a warp spread over the banks.
__global__ void __launch_bounds__(kThreads) chol_solve_kernel(const double *__restrict__ H,
                                                              const double *__restrict__ g, int d,
                                                              const double *__restrict__ x, double *x_next,
                                                              double *scratch, int *status, int use_smem) {
  extern __shared__ double sm[];
  const int lda = d + 1;
  double *a = use_smem ? sm : scratch;                                 // d x lda, lower triangle used
  double *z = use_smem ? sm + (size_t)d * lda : scratch + (size_t)d * lda;  // d
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;          // 32 x 16 thread grid
  constexpr int kRows = kThreads / 32;
  for (int i = ty; i < d; i += kRows)
    for (int c = tx; c <= i; c += 32) a[(int64_t)i * lda + c] = H[(int64_t)i * d + c];
  for (int i = tid; i < d; i += kThreads) z[i] = g[i];
  __syncthreads();
  bool bad = false;
  for (int j = 0; j < d; ++j) {
    const double piv = a[(int64_t)j * lda + j];
    if (!(piv > 0.0)) {  // every thread reads the same pivot: uniform exit
      bad = true;
      break;
    }
    const double rinv = 1.0 / piv;
    for (int i = j + 1 + ty; i < d; i += kRows) {
      const double aij = a[(int64_t)i * lda + j] * rinv;
      double *ai = a + (int64_t)i * lda;
      for (int c = j + 1 + tx; c <= i; c += 32) ai[c] -= aij * a[(int64_t)c * lda + j];
    }
    __syncthreads();
  }
  if (bad) {
    for (int i = tid; i < d; i += kThreads) x_next[i] = x[i];
    if (tid == 0) set_status(status, 3 /* IHS_ERR_NOT_SPD */);
    return;
  }
  // L_ij = a_ij / sqrt(a_jj), L_jj = sqrt(a_jj)
  for (int i = ty; i < d; i += kRows)
    for (int c = tx; c < i; c += 32) a[(int64_t)i * lda + c] /= sqrt(a[(int64_t)c * lda + c]);
  __syncthreads();
  for (int i = tid; i < d; i += kThreads) a[(int64_t)i * lda + i] = sqrt(a[(int64_t)i * lda + i]);
  __syncthreads();
  if (tid < 32) {
    const int lane = tid;
    // forward: L y = g (column-oriented; row i subtracts terms j = 0..i-1 in order)
    for (int j = 0; j < d; ++j) {
      __syncwarp();
      const double yj = z[j] / a[(int64_t)j * lda + j];
      __syncwarp();
      if (lane == 0) z[j] = yj;
      for (int i = j + 1 + lane; i < d; i += 32) z[i] -= a[(int64_t)i * lda + j] * yj;
    }
    // backward: L^T u = y
    for (int i = d - 1; i >= 0; --i) {
      __syncwarp();
      const double ui = z[i] / a[(int64_t)i * lda + i];
      __syncwarp();
      if (lane == 0) z[i] = ui;
      for (int k = lane; k < i; k += 32) z[k] -= a[(int64_t)i * lda + k] * ui;
    }
    __syncwarp();
    for (int i = lane; i < d; i += 32) x_next[i] = x[i] + z[i];
  }
}

// d <= 32*S (and <= 16*R): thread (ty, tx) of a 16 x 32 grid keeps the lower-
// triangle elements (ty + 16r, tx + 32s) in REGISTERS for the whole
// factorisation.  Step j: the owners of column j publish it through a
// double-buffered shared vector (one barrier per column); every thread then
// applies a_ic -= a_ij a_cj / a_jj to its elements with c > j.  The unscaled
// columns are also kept in shared memory; a final pass scales them to
// L_ij = a_ij / sqrt(a_jj).  The two triangular solves run in warp 0 with the
// right-hand side in registers and one shuffle per step.
template <int R, int S>
__global__ void __launch_bounds__(kThreads) chol_reg_kernel(const double *__restrict__ H,
                                                            const double *__restrict__ g, int d,
                                                            const double *__restrict__ x, double *x_next,
                                                            int *status) {
  static_assert(16 * R >= 32 * S || true, "");
  extern __shared__ double sm[];
  const int lda = d + 1;
  double *L = sm;                          // d x lda: unscaled columns, then L
  double *colbuf = sm + (size_t)d * lda;   // 2 x (32 S)
  double *rdiag = colbuf + 2 * 32 * S;     // 32 S: 1 / L_jj
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
  double a[R][S];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int i = ty + 16 * r, c = tx + 32 * s;
      a[r][s] = (i < d && c <= i) ? H[(int64_t)i * d + c] : 0.0;
    }
  bool bad = false;
  for (int j = 0; j < d; ++j) {
    const int js = j >> 5, jt = j & 31;
    double *cb = colbuf + (j & 1) * 32 * S;
    if (tx == jt) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int i = ty + 16 * r;
        if (i >= j && i < d) {
          double v = 0.0;
#pragma unroll
          for (int s = 0; s < S; ++s)
            if (s == js) v = a[r][s];
          cb[i] = v;
          L[(int64_t)i * lda + j] = v;
        }
      }
    }
    __syncthreads();
    const double piv = cb[j];
    if (!(piv > 0.0)) {
      bad = true;
      break;
    }
    const double rinv = 1.0 / piv;
    double ci[R], cc[S];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = ty + 16 * r;
      ci[r] = (i > j && i < d) ? cb[i] * rinv : 0.0;
    }
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int c = tx + 32 * s;
      cc[s] = (c > j && c < d) ? cb[c] : 0.0;
    }
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int s = 0; s < S; ++s) a[r][s] -= ci[r] * cc[s];
  }
  if (bad) {
    for (int i = tid; i < d; i += kThreads) x_next[i] = x[i];
    if (tid == 0) set_status(status, 3 /* IHS_ERR_NOT_SPD */);
    return;
  }
  // (elements above the diagonal in a[][] picked up garbage products above; they are never read)
  __syncthreads();
  for (int j = tid; j < d; j += kThreads) rdiag[j] = 1.0 / sqrt(L[(int64_t)j * lda + j]);
  __syncthreads();
  for (int i = ty; i < d; i += 16)
    for (int c = tx; c <= i; c += 32)
      L[(int64_t)i * lda + c] = (c == i) ? sqrt(L[(int64_t)i * lda + i]) : L[(int64_t)i * lda + c] * rdiag[c];
  __syncthreads();
  if (tid < 32) {
    const int lane = tid;
    double z[S];
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int i = lane + 32 * s;
      z[s] = i < d ? g[i] : 0.0;
    }
    // forward: L y = g
#pragma unroll
    for (int s = 0; s < S; ++s) {
      for (int jj = 0; jj < 32; ++jj) {
        const int j = 32 * s + jj;
        if (j >= d) break;
        const double yj = __shfl_sync(0xffffffffu, z[s], jj) * rdiag[j];
        if (lane == jj) z[s] = yj;
#pragma unroll
        for (int q = s; q < S; ++q) {
          const int i = lane + 32 * q;
          if (i > j && i < d) z[q] -= L[(int64_t)i * lda + j] * yj;
        }
      }
    }
    // backward: L^T u = y
#pragma unroll
    for (int s = S - 1; s >= 0; --s) {
      for (int jj = 31; jj >= 0; --jj) {
        const int i = 32 * s + jj;
        if (i >= d) continue;
        const double ui = __shfl_sync(0xffffffffu, z[s], jj) * rdiag[i];
        if (lane == jj) z[s] = ui;
#pragma unroll
        for (int q = 0; q <= s; ++q) {
          const int k = lane + 32 * q;
          if (k < i) z[q] -= L[(int64_t)i * lda + k] * ui;
        }
      }
    }
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int i = lane + 32 * s;
      if (i < d) x_next[i] = x[i] + z[s];
    }
  }
}

template <int R, int S>
void launch_reg(const double *H, const double *g, int d, const double *x, double *x_next, int *status,
                cudaStream_t st) {
  const size_t smem = ((size_t)d * (d + 1) + 3 * 32 * S) * 8;
  IHS_SMEM_ATTR((chol_reg_kernel<R, S>), smem);
  chol_reg_kernel<R, S><<<1, kThreads, smem, st>>>(H, g, d, x, x_next, status);
}

// ----------------------------------------------------------------------------
// Blocked right-looking Cholesky in one CTA for D = ceil(d/32)*32 <= 160 (the
// matrix is padded with an identity block).  Per 32-column block kb:
//   1. warp 0 factors the 32x32 diagonal block in registers (lane i holds row
//      i; one shuffle broadcasts each column), storing L11 and 1/L_jj;
//   2. the rows below solve X L11^T = A21 (one thread per row, L11 broadcast
//      from shared memory);
//   3. the trailing lower triangle is updated A22 -= L21 L21^T on the DMMA pipe
//      (mma.sync m8n8k4 f64, 8x8 tiles spread over the 16 warps).
// Then warp 0 runs both triangular solves with the right-hand side in
// registers.  Leading dimension D + 4 (== 4 mod 16 doubles) keeps the DMMA
// fragment loads conflict-free.
__device__ __forceinline__ void dmma884(double &c0, double &c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}


// Compile-time unrolled column steps (template recursion keeps row[] in registers).
template <int J>
__device__ __forceinline__ void diag_step(double (&row)[32], int lane, bool &bad, double *rd) {
  const double piv = __shfl_sync(0xffffffffu, row[J], J);
  bad |= !(piv > 0.0);
  const double sq = sqrt(piv);
  const double r = 1.0 / sq;
  const double lij = (lane > J) ? row[J] * r : (lane == J ? sq : 0.0);
  row[J] = lij;
  if (lane == 0) rd[J] = r;
#pragma unroll
  for (int k = J + 1; k < 32; ++k) {
    const double lkj = __shfl_sync(0xffffffffu, lij, k);
    if (lane >= k) row[k] -= lij * lkj;
  }
}
template <int... Js>
__device__ __forceinline__ void diag_steps(double (&row)[32], int lane, bool &bad, double *rd,
                                           std::integer_sequence<int, Js...>) {
  (diag_step<Js>(row, lane, bad, rd), ...);
}
template <int J>
__device__ __forceinline__ void trsm_step(double (&xr)[32], const double *rd, const double *L11, int lda) {
  const double xj = xr[J] * rd[J];
  xr[J] = xj;
#pragma unroll
  for (int k = J + 1; k < 32; ++k) xr[k] -= xj * L11[k * lda + J];
}
template <int... Js>
__device__ __forceinline__ void trsm_steps(double (&xr)[32], const double *rd, const double *L11, int lda,
                                           std::integer_sequence<int, Js...>) {
  (trsm_step<Js>(xr, rd, L11, lda), ...);
}

constexpr int kBThreads = 256;
template <int NBLK>
__global__ void __launch_bounds__(kBThreads) chol_blocked_kernel(const double *__restrict__ H,
                                                                const double *__restrict__ g, int d,
                                                                const double *__restrict__ x, double *x_next,
                                                                int *status) {
  constexpr int D = 32 * NBLK;
  constexpr int lda = D + 4;
  extern __shared__ double sm[];
  double *Ls = sm;               // D x lda
  double *rdiag = sm + D * lda;  // D
  __shared__ int s_bad;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = warp; i < D; i += kBThreads / 32)
    for (int c = lane; c <= i; c += 32)
      Ls[i * lda + c] = (i < d) ? H[(int64_t)i * d + c] : (c == i ? 1.0 : 0.0);
  if (tid == 0) s_bad = 0;
  __syncthreads();
#pragma unroll 1
  for (int kb = 0; kb < D; kb += 32) {
    // 1. diagonal block
    if (warp == 0) {
      double row[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) row[c] = (c <= lane) ? Ls[(kb + lane) * lda + kb + c] : 0.0;
      bool bad = false;
      diag_steps(row, lane, bad, rdiag + kb, std::make_integer_sequence<int, 32>{});
      if (bad && lane == 0) s_bad = 1;
#pragma unroll
      for (int c = 0; c < 32; ++c)
        if (c <= lane) Ls[(kb + lane) * lda + kb + c] = row[c];
    }
    __syncthreads();
    if (s_bad) break;
    // 2. panel: rows below solve X L11^T = A21
    const int nbelow = D - kb - 32;
    if (tid < nbelow) {
      const int i = kb + 32 + tid;
      double xr[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) xr[c] = Ls[i * lda + kb + c];
      trsm_steps(xr, rdiag + kb, Ls + kb * lda + kb, lda, std::make_integer_sequence<int, 32>{});
#pragma unroll
      for (int c = 0; c < 32; ++c) Ls[i * lda + kb + c] = xr[c];
    }
    __syncthreads();
    // 3. trailing update A22 -= L21 L21^T (lower 8x8 tiles on DMMA)
    if (nbelow > 0) {
      const int nt = nbelow / 8;
      const int ntri = nt * (nt + 1) / 2;
      for (int t = warp; t < ntri; t += kBThreads / 32) {
        int ti = 0, rem = t;  // row-major enumeration of {(ti, tj): tj <= ti}
        while (rem > ti) {
          rem -= ti + 1;
          ++ti;
        }
        const int tj = rem;
        const int I = kb + 32 + 8 * ti, J = kb + 32 + 8 * tj;
        double c0 = 0.0, c1 = 0.0;
#pragma unroll
        for (int kk = 0; kk < 32; kk += 4) {
          const double a = Ls[(I + (lane >> 2)) * lda + kb + kk + (lane & 3)];
          const double b = Ls[(J + (lane >> 2)) * lda + kb + kk + (lane & 3)];
          dmma884(c0, c1, a, b);
        }
        const int r = I + (lane >> 2), c = J + 2 * (lane & 3);
        Ls[r * lda + c] -= c0;
        Ls[r * lda + c + 1] -= c1;
      }
    }
    __syncthreads();
  }
  if (s_bad) {
    for (int i = tid; i < d; i += kBThreads) x_next[i] = x[i];
    if (tid == 0) set_status(status, 3 /* IHS_ERR_NOT_SPD */);
    return;
  }
  if (warp == 0) {
    double z[NBLK];
#pragma unroll
    for (int s = 0; s < NBLK; ++s) {
      const int i = lane + 32 * s;
      z[s] = i < d ? g[i] : 0.0;
    }
    // forward: L y = g
#pragma unroll
    for (int s = 0; s < NBLK; ++s) {
#pragma unroll 4
      for (int jj = 0; jj < 32; ++jj) {
        const int j = 32 * s + jj;
        const double yj = __shfl_sync(0xffffffffu, z[s], jj) * rdiag[j];
        if (lane == jj) z[s] = yj;
#pragma unroll
        for (int q = s; q < NBLK; ++q) {
          const int i = lane + 32 * q;
          if (i > j) z[q] -= Ls[i * lda + j] * yj;
        }
      }
    }
    // backward: L^T u = y
#pragma unroll
    for (int s = NBLK - 1; s >= 0; --s) {
#pragma unroll 4
      for (int jj = 31; jj >= 0; --jj) {
        const int i = 32 * s + jj;
        const double ui = __shfl_sync(0xffffffffu, z[s], jj) * rdiag[i];
        if (lane == jj) z[s] = ui;
#pragma unroll
        for (int q = 0; q <= s; ++q) {
          const int k = lane + 32 * q;
          if (k < i) z[q] -= Ls[i * lda + k] * ui;
        }
      }
    }
#pragma unroll
    for (int s = 0; s < NBLK; ++s) {
      const int i = lane + 32 * s;
      if (i < d) x_next[i] = x[i] + z[s];
    }
  }
}

template <int NBLK>
void launch_blocked(const double *H, const double *g, int d, const double *x, double *x_next, int *status,
                    cudaStream_t st) {
  constexpr int D = 32 * NBLK;
  const size_t smem = ((size_t)D * (D + 4) + D) * 8;
  IHS_SMEM_ATTR((chol_blocked_kernel<NBLK>), smem);
  chol_blocked_kernel<NBLK><<<1, kBThreads, smem, st>>>(H, g, d, x, x_next, status);
}
}  // namespace

size_t chol_scratch_bytes(int64_t d) { return (size_t)(d * (d + 1) + d) * 8; }

cudaError_t launch_ols_update(const double *H, const double *g, int64_t d, const double *x, double *x_next,
                              double *scratch, int *status, int num_sms, cudaStream_t st, LaunchCounter lc) {
  (void)num_sms;
  if (d <= 160) {
    const int nblk = (int)((d + 31) / 32);
    switch (nblk) {
      case 1: launch_blocked<1>(H, g, (int)d, x, x_next, status, st); break;
      case 2: launch_blocked<2>(H, g, (int)d, x, x_next, status, st); break;
      case 3: launch_blocked<3>(H, g, (int)d, x, x_next, status, st); break;
      case 4: launch_blocked<4>(H, g, (int)d, x, x_next, status, st); break;
      default: launch_blocked<5>(H, g, (int)d, x, x_next, status, st); break;
    }
    lc.add();
    return cudaGetLastError();
  }
  const size_t need = (size_t)(d * (d + 1) + d) * 8;
  const int use_smem = need <= kSmemLimit;
  const size_t smem = use_smem ? need : 0;
  IHS_SMEM_ATTR(chol_solve_kernel, smem);
  chol_solve_kernel<<<1, kThreads, smem, st>>>(H, g, (int)d, x, x_next, scratch, status, use_smem);
  lc.add();
  return cudaGetLastError();
}

}  // namespace ihs
