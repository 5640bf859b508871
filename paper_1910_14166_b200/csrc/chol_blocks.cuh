// Building blocks of the blocked Cholesky (a6, OLS step; PAPER.md:83-86,
// T_solve = O(d^3)): the 32x32 diagonal-block factorisation
// (one warp) and the 32-column triangular solve of the rows below (one thread
// per row), both with the row in registers and the 32 column steps unrolled at
// compile time.  Measured on B200 (tools/probe/chol_probe.cu, clocks per
// call): 7.1k (factor, column broadcast through shared memory; 10.4k with
// shuffles) / 2.8k (solve, 128 rows) vs 16.4k / 10.8k for a rolled variant
// that rotates the register row; the fp64 latencies on the column chain are
// DFMA 23, rsqrt 65, shuffle ~27 clocks.
#pragma once
#include <utility>

#include "common.cuh"

namespace ihs {

namespace chol_detail {
// Column step J: l_J = row[J] / sqrt(pivot); the column is published through
// shared memory (one store per lane, double-buffered by step parity) and the
// rank-1 update reads it back as broadcasts -- measured 7.1k clocks per 32x32
// factorisation vs 10.4k with one shuffle per updated column.
template <int J>
__device__ __forceinline__ void diag_step(double (&row)[32], int lane, bool &bad, double *rd, int jcheck,
                                          double *col) {
  const double piv = __shfl_sync(0xffffffffu, row[J], J);
  bad |= (J < jcheck) && !(piv > 0.0);
  double ljj, r;
  pivot_rsqrt(piv, ljj, r);
  const double lij = (lane > J) ? row[J] * r : (lane == J ? ljj : 0.0);
  row[J] = lij;
  if (lane == 0) rd[J] = r;
  col[(J & 1) * 32 + lane] = lij;
  __syncwarp();
#pragma unroll
  for (int k = J + 1; k < 32; ++k) row[k] = fma(-lij, col[(J & 1) * 32 + k], row[k]);
}
template <int... Js>
__device__ __forceinline__ void diag_steps(double (&row)[32], int lane, bool &bad, double *rd, int jcheck,
                                           double *col, std::integer_sequence<int, Js...>) {
  (diag_step<Js>(row, lane, bad, rd, jcheck, col), ...);
}
template <int J>
__device__ __forceinline__ void trsm_step(double (&xr)[32], const double *rd, const double *L11, int ld) {
  const double xj = xr[J] * rd[J];
  xr[J] = xj;
#pragma unroll
  for (int k = J + 1; k < 32; ++k) xr[k] -= xj * L11[k * ld + J];
}
template <int... Js>
__device__ __forceinline__ void trsm_steps(double (&xr)[32], const double *rd, const double *L11, int ld,
                                           std::integer_sequence<int, Js...>) {
  (trsm_step<Js>(xr, rd, L11, ld), ...);
}
}  // namespace chol_detail

// One warp factors the 32x32 lower block B (row-major, leading dimension ld)
// in place, B = L L^T; rd[j] = 1 / L_jj.  Lane i holds row i; col is 64
// doubles of shared scratch for the column broadcasts.  Entries right of the
// diagonal pick up values that are never read.  Returns (in every lane)
// whether a pivot <= 0 was met among columns j < jcheck.
__device__ __forceinline__ bool warp_chol32(double *B, int ld, double *rd, int jcheck, double *col) {
  const int lane = threadIdx.x & 31;
  double row[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) row[c] = (c <= lane) ? B[lane * ld + c] : 0.0;
  bool bad = false;
  chol_detail::diag_steps(row, lane, bad, rd, jcheck, col, std::make_integer_sequence<int, 32>{});
#pragma unroll
  for (int c = 0; c < 32; ++c)
    if (c <= lane) B[lane * ld + c] = row[c];
  return __any_sync(0xffffffffu, bad);
}

// One thread solves x L11^T = a for its own 32-wide row segment R (in place):
// x_j = (a_j - sum_{k<j} x_k L_jk) / L_jj.  L11 is the factored 32x32 block
// (row-major, leading dimension ld; read as broadcasts), rd its reciprocal
// diagonal.
__device__ __forceinline__ void thread_trsm32(double *R, const double *L11, int ld, const double *rd) {
  double xr[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) xr[c] = R[c];
  chol_detail::trsm_steps(xr, rd, L11, ld, std::make_integer_sequence<int, 32>{});
#pragma unroll
  for (int c = 0; c < 32; ++c) R[c] = xr[c];
}

}  // namespace ihs
