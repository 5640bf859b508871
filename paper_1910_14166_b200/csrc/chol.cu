// a6, OLS: x^{t+1} = x^t + H^{-1} g (Eq. (2) with C = R^d, PAPER.md:83-86;
// T_solve = O(d^3)).  d <= 160: blocked Cholesky H = L L^T
// in one CTA with H in shared memory (this file); d > 160: multi-CTA panel
// factorisation (chol_large.cu).  A pivot <= 0 sets IHS_ERR_NOT_SPD (reading
// R13) and x_next = x.  Latency-bound: O(d) dependent column steps.
#include "common.cuh"
#include "kernels.h"
#include "chol_blocks.cuh"

#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>


namespace ihs {

namespace {
// ----------------------------------------------------------------------------
// Blocked right-looking Cholesky in one CTA for D = ceil(d/32)*32 <= 160 (the
// matrix is padded with an identity block).  Per 32-column block kb:
//   1. warp 0 factors the 32x32 diagonal block in registers (warp_chol32:
//      lane i holds row i; one shuffle broadcasts each column), storing L11
//      and 1/L_jj;
//   2. the rows below solve X L11^T = A21 (thread_trsm32: one thread per row,
//      L11 broadcast from shared memory);
//   3. the trailing lower triangle is updated A22 -= L21 L21^T on the DMMA pipe
//      (mma.sync m8n8k4 f64, 8x8 tiles spread over the 16 warps).
// g rides along as an augmented row (the forward solve comes out of the
// factorisation); then warp 0 runs the backward solve in registers.  Leading dimension D + 4 (== 4 mod 16 doubles) keeps the DMMA
// fragment loads conflict-free.
__device__ __forceinline__ void dmma884(double &c0, double &c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}


constexpr int kBThreads = 256;
// The right-hand side rides along as row D of an augmented matrix [[H, 0], [g^T, 0]]
// (rows D+1..D+7 are zero so the DMMA trailing update keeps whole 8-row tiles):
// the panel TRSM and the trailing updates turn row D into y = L^{-1} g, so only
// the backward solve L^T u = y runs after the factorisation.
// The factorisation and solves on the loaded augmented Ls (shared memory), by
// the whole CTA of kBThreads threads: shared by chol_blocked_kernel (H from
// global) and gram_ols_kernel (H reduced from a cluster's Gram partials).
// Factorisation only: Ls holds L (lower triangle) and rdiag[j] = 1 / L_jj on
// return; true (for every thread) if a pivot was not positive.
template <int NBLK>
__device__ __forceinline__ bool chol_factor_body(double *Ls, double *rdiag, double *colbuf, int &s_bad) {
  constexpr int D = 32 * NBLK;
  constexpr int lda = D + 4;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_bad = 0;
  __syncthreads();
#pragma unroll 1
  for (int kb = 0; kb < D; kb += 32) {
    // 1. diagonal block
    if (warp == 0) {
      const bool bad = warp_chol32(Ls + kb * lda + kb, lda, rdiag + kb, 32, colbuf);
      if (bad && lane == 0) s_bad = 1;
    }
    __syncthreads();
    if (s_bad) break;
    // 2. panel: rows below (incl. the g row) solve X L11^T = A21
    const int nbelow = D - kb - 32;
    if (tid < nbelow + 8) thread_trsm32(Ls + (kb + 32 + tid) * lda + kb, Ls + kb * lda + kb, lda, rdiag + kb);
    __syncthreads();
    // 3. trailing update A22 -= L21 L21^T (lower 8x8 tiles on DMMA), plus the
    //    g-row tile against every trailing column tile
    const int nt = nbelow / 8;
    const int ntri = nt * (nt + 1) / 2;
    for (int t = warp; t < ntri + nt; t += kBThreads / 32) {
      int ti, tj;
      if (t < ntri) {
        ti = 0;
        int rem = t;  // row-major enumeration of {(ti, tj): tj <= ti}
        while (rem > ti) {
          rem -= ti + 1;
          ++ti;
        }
        tj = rem;
      } else {
        ti = nt;
        tj = t - ntri;
      }
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
    __syncthreads();
  }
  return s_bad != 0;
}

template <int NBLK>
__device__ __forceinline__ void chol_blocked_body(double *Ls, double *rdiag, double *colbuf, int &s_bad, int d,
                                                  const double *__restrict__ x, double *x_next, int *status) {
  constexpr int D = 32 * NBLK;
  constexpr int lda = D + 4;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (chol_factor_body<NBLK>(Ls, rdiag, colbuf, s_bad)) {
    for (int i = tid; i < d; i += kBThreads) x_next[i] = x[i];
    if (tid == 0) set_status(status, 3 /* IHS_ERR_NOT_SPD */);
    return;
  }
  if (warp == 0) {
    // backward: L^T u = y, y = row D
    double z[NBLK];
#pragma unroll
    for (int s = 0; s < NBLK; ++s) z[s] = Ls[D * lda + lane + 32 * s];
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

// H^{-1} = L^{-T} L^{-1} from the factor in Ls / rdiag (the look-ahead OLS
// factor, api.cu), with Y = L^{-1} kept TRANSPOSED in the unused upper
// triangle of Ls (Ls[a][b] = Y[b][a] for a < b; Y's diagonal is rdiag), so no
// extra shared memory beyond one 32 x 36 buffer per column block:
//   A. warp I inverts the diagonal block L_II (lane c owns column c of Y_II in
//      registers; the L row is a broadcast; 32 x 32 fully unrolled);
//   B. row blocks I = 1.. in order: T_IJ = sum_{K=J}^{I-1} L_IK Y_KJ, then
//      Y_IJ = -Y_II T_IJ (DMMA m8n8k4 f64, 8x8 tiles over the 8 warps);
//   C. Hinv = Y^T Y, lower 8x8 tiles on DMMA, both halves written to global.
// Both operands of every DMMA are rows of Ls at leading dimension D + 4, the
// conflict-free fragment pattern of the factorisation.  (A thread-per-column
// forward substitution on packed rows took ~200 us at d = 128; this ~10 us.)
template <int NBLK>
__device__ __forceinline__ double yT(const double *Ls, const double *rdiag, int a, int b) {
  constexpr int lda = 32 * NBLK + 4;  // Y[b][a]: upper storage, diagonal in rdiag, zero above
  return b > a ? Ls[a * lda + b] : (b == a ? rdiag[a] : 0.0);
}

template <int NBLK>
__device__ __forceinline__ void chol_inverse_body(double *Ls, const double *rdiag, double *Tt, int d,
                                                  double *__restrict__ Hinv) {
  constexpr int D = 32 * NBLK;
  constexpr int lda = D + 4;
  constexpr int ldt = 36;  // Tt: per J, 32 x ldt (T transposed)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // A. diagonal blocks
  if (warp < NBLK) {
    const int I0 = 32 * warp, c = lane;
    double y[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      double s = (i == c) ? 1.0 : 0.0;
#pragma unroll
      for (int k = 0; k < i; ++k) s = fma(-Ls[(I0 + i) * lda + I0 + k], y[k], s);
      y[i] = s * rdiag[I0 + i];
    }
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (i > c) Ls[(I0 + c) * lda + I0 + i] = y[i];
  }
  __syncthreads();
  const int r4 = lane >> 2, k4 = lane & 3;
  // B. off-diagonal blocks, row block by row block
#pragma unroll 1
  for (int I = 1; I < NBLK; ++I) {
    // T_IJ (J < I): 16 tiles each
    for (int t = warp; t < 16 * I; t += kBThreads / 32) {
      const int J = t >> 4, ti = (t >> 2) & 3, tn = t & 3;
      const int R = 32 * I + 8 * ti, N = 32 * J + 8 * tn;
      double c0 = 0.0, c1 = 0.0;
      for (int k0 = 32 * J; k0 < 32 * I; k0 += 4) {
        const double a = Ls[(R + r4) * lda + k0 + k4];            // L[R + r][k]
        const double b = yT<NBLK>(Ls, rdiag, N + r4, k0 + k4);     // Y[k][N + n]
        dmma884(c0, c1, a, b);
      }
      double *T = Tt + J * 32 * ldt;  // T[r][n] stored at Tt[n][r]
      const int r = 8 * ti + r4, n = 8 * tn + 2 * k4;
      T[n * ldt + r] = c0;
      T[(n + 1) * ldt + r] = c1;
    }
    __syncthreads();
    // Y_IJ = -Y_II T_IJ, stored transposed into Ls[32J + n][32I + r]
    for (int t = warp; t < 16 * I; t += kBThreads / 32) {
      const int J = t >> 4, ti = (t >> 2) & 3, tn = t & 3;
      const double *T = Tt + J * 32 * ldt;
      double c0 = 0.0, c1 = 0.0;
#pragma unroll
      for (int k0 = 0; k0 < 32; k0 += 4) {
        const double a = yT<NBLK>(Ls, rdiag, 32 * I + k0 + k4, 32 * I + 8 * ti + r4);  // Y_II[r][k]
        const double b = T[(8 * tn + r4) * ldt + k0 + k4];                           // T[k][n]
        dmma884(c0, c1, a, b);
      }
      const int r = 32 * I + 8 * ti + r4, n = 32 * J + 8 * tn + 2 * k4;
      Ls[n * lda + r] = -c0;
      Ls[(n + 1) * lda + r] = -c1;
    }
    __syncthreads();
  }
  // C. Hinv[p][q] = sum_{k >= p} Y[k][p] Y[k][q], lower 8x8 tiles (tp >= tq)
  constexpr int NT8 = D / 8;
  for (int t = warp; t < NT8 * (NT8 + 1) / 2; t += kBThreads / 32) {
    int tp = 0, rem = t;
    while (rem > tp) {
      rem -= tp + 1;
      ++tp;
    }
    const int tq = rem, P0 = 8 * tp, Q0 = 8 * tq;
    if (P0 >= d) continue;
    double c0 = 0.0, c1 = 0.0;
    for (int k0 = P0; k0 < D; k0 += 4) {
      const double a = yT<NBLK>(Ls, rdiag, P0 + r4, k0 + k4);  // Y[k][p]
      const double b = yT<NBLK>(Ls, rdiag, Q0 + r4, k0 + k4);  // Y[k][q]
      dmma884(c0, c1, a, b);
    }
    const int p = P0 + r4, q = Q0 + 2 * k4;
    if (p < d) {
      if (q < d) {
        Hinv[(int64_t)p * d + q] = c0;
        Hinv[(int64_t)q * d + p] = c0;
      }
      if (q + 1 < d) {
        Hinv[(int64_t)p * d + q + 1] = c1;
        Hinv[(int64_t)(q + 1) * d + p] = c1;
      }
    }
  }
}

template <int NBLK>
__global__ void __launch_bounds__(kBThreads) chol_blocked_kernel(const double *__restrict__ H,
                                                                const double *__restrict__ g, int d,
                                                                const double *__restrict__ x, double *x_next,
                                                                int *status, const int *run) {
  if (run && *run == 0) return;  // the CG solve before it finished
  constexpr int D = 32 * NBLK;
  constexpr int DA = D + 8;  // rows incl. the augmented g row and its zero tile padding
  constexpr int lda = D + 4;
  extern __shared__ double sm[];
  double *Ls = sm;                // DA x lda
  double *rdiag = sm + DA * lda;  // D
  __shared__ int s_bad;
  __shared__ double colbuf[64];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // lower triangle of H (identity padding), 16 loads in flight per thread
  constexpr int PER = D * D / kBThreads;
#pragma unroll 1
  for (int k0 = 0; k0 < PER; k0 += 16) {
    double v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int e = tid + (k0 + k) * kBThreads, i = e / D, c = e % D;
      v[k] = (k0 + k < PER && c <= i) ? ((i < d) ? H[(int64_t)i * d + c] : (c == i ? 1.0 : 0.0)) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int e = tid + (k0 + k) * kBThreads, i = e / D, c = e % D;
      if (k0 + k < PER && c <= i) Ls[i * lda + c] = v[k];
    }
  }
  for (int i = D + warp; i < DA; i += kBThreads / 32)
    for (int c = lane; c < D; c += 32) Ls[i * lda + c] = (i == D && c < d) ? g[c] : 0.0;
  chol_blocked_body<NBLK>(Ls, rdiag, colbuf, s_bad, d, x, x_next, status);
}

// ---------------------------------------------------------------------------
// a4 + a6 fused for d <= 128 (OLS): one thread-block cluster.  CTAs 1..CL-1
// form Gram partials of row ranges of SA on DMMA (mma.sync m8n8k4 f64, 32x32
// warp tiles over the full D x D); after a cluster barrier each of them sums a
// slice of the lower triangle over all partials in CTA order (DSMEM reads) and
// stores it straight into CTA 0's augmented Cholesky matrix (DSMEM writes);
// after a second barrier CTA 0 factorises and solves (chol_blocked_body).
// Replaces the Gram launch pair + the Cholesky launch (one launch, H never
// round-trips through L2 on the critical path; H_out, if given, gets a copy).
constexpr int kGoRows = 64;  // SA rows per staging chunk
// INV (the look-ahead factor, api.cu): no right-hand side; CTA 0 factorises
// and writes H^{-1} to Hinv (zeros and IHS_ERR_NOT_SPD on a non-positive pivot).
template <int NBLK, bool INV>
__global__ void __launch_bounds__(kBThreads, 1) gram_ols_kernel(const double *__restrict__ SA, int64_t m, int d,
                                                               double scale2, const double *__restrict__ g,
                                                               const double *__restrict__ x, double *x_next,
                                                               double *H_out, int *status, double *Hinv) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  constexpr int D = 32 * NBLK;
  constexpr int DA = D + 8;
  constexpr int lda = D + 4;      // Cholesky layout (CTA 0)
  constexpr int lds = D + 4;      // staging stride (== 4 mod 16: conflict-free fragments)
  constexpr int NT = NBLK * NBLK;  // 32x32 warp tiles of the full D x D
  extern __shared__ double sm[];
  __shared__ int s_bad;
  __shared__ double colbuf[64];
  const int rank = (int)cluster.block_rank(), cs = (int)cluster.num_blocks();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (rank == 0) {
    double *Ls = sm;
    for (int i = warp; i < DA; i += kBThreads / 32) {
      if (i < D) {
        if (i >= d)  // identity padding; the lower triangle of H arrives from the reducers
          for (int c = lane; c <= i; c += 32) Ls[i * lda + c] = (c == i ? 1.0 : 0.0);
      } else {
        for (int c = lane; c < D; c += 32) Ls[i * lda + c] = (!INV && i == D && c < d) ? g[c] : 0.0;
      }
    }
  } else {
    double *S = sm;                          // kGoRows x lds
    double *Hp = sm + kGoRows * lds;         // D x D partial
    const int64_t nw = cs - 1, w0 = rank - 1;
    const int64_t r0 = m * w0 / nw, r1 = m * (w0 + 1) / nw;
    double acc[2][4][4][2];
#pragma unroll
    for (int t = 0; t < 2; ++t)
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[t][i][j][0] = acc[t][i][j][1] = 0.0;
    for (int64_t rb = r0; rb < r1; rb += kGoRows) {
      const int rows = (int)min((int64_t)kGoRows, r1 - rb);
      __syncthreads();  // the previous chunk's fragments are consumed
      // all loads of the chunk in flight before the stores (a runtime-bounded
      // loop issued one L2 round trip at a time: the factor took 0.35 ms
      // beside a gather)
      constexpr int PER = kGoRows * D / kBThreads;
      double v[PER];
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        const int e = tid + k * kBThreads, r = e / D, c = e % D;
        v[k] = (r < rows && c < d) ? SA[(rb + r) * d + c] : 0.0;
      }
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        const int e = tid + k * kBThreads;
        S[(e / D) * lds + e % D] = v[k];
      }
      __syncthreads();
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int tile = warp + 8 * t;
        if (tile < NT) {
          const int I = 32 * (tile / NBLK), J = 32 * (tile % NBLK);
#pragma unroll 4
          for (int kk = 0; kk < kGoRows; kk += 4) {
            const int kr = kk + (lane & 3);
            double a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = S[kr * lds + I + 8 * i + (lane >> 2)];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = S[kr * lds + J + 8 * j + (lane >> 2)];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
              for (int j = 0; j < 4; ++j) dmma884(acc[t][i][j][0], acc[t][i][j][1], a[i], b[j]);
          }
        }
      }
    }
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const int tile = warp + 8 * t;
      if (tile < NT) {
        const int I = 32 * (tile / NBLK), J = 32 * (tile % NBLK);
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int r = I + 8 * i + (lane >> 2), c = J + 8 * j + 2 * (lane & 3);
            Hp[r * D + c] = acc[t][i][j][0];
            Hp[r * D + c + 1] = acc[t][i][j][1];
          }
      }
    }
  }
  cluster.sync();
  if (rank > 0) {
    // reduce a slice of the lower triangle over the partials (CTA order) into CTA 0
    double *Ls0 = cluster.map_shared_rank(sm, 0);
    const int nw = cs - 1;
    const double *parts[15];
#pragma unroll
    for (int r = 1; r < 16; ++r) parts[r - 1] = cluster.map_shared_rank(sm + kGoRows * lds, r < cs ? r : 1);
    for (int e = (rank - 1) * kBThreads + tid; e < D * D; e += nw * kBThreads) {
      const int i = e / D, j = e % D;
      if (j > i || i >= d) continue;
      double u[15];  // the cs - 1 DSMEM loads in flight, then added in CTA order
#pragma unroll
      for (int r = 1; r < 16; ++r) u[r - 1] = (r < cs) ? parts[r - 1][e] : 0.0;
      double v = 0.0;
#pragma unroll
      for (int r = 1; r < 16; ++r)
        if (r < cs) v += u[r - 1];
      v *= scale2;
      Ls0[i * lda + j] = v;
      if (H_out) {
        H_out[(int64_t)i * d + j] = v;
        H_out[(int64_t)j * d + i] = v;
      }
    }
  }
  cluster.sync();
  if (rank != 0) return;
  if constexpr (INV) {
    if (chol_factor_body<NBLK>(sm, sm + DA * lda, colbuf, s_bad)) {
      for (int e = tid; e < d * d; e += kBThreads) Hinv[e] = 0.0;
      if (tid == 0) set_status(status, 3 /* IHS_ERR_NOT_SPD */);
      return;
    }
    chol_inverse_body<NBLK>(sm, sm + DA * lda, sm + DA * lda + D, d, Hinv);
  } else {
    chol_blocked_body<NBLK>(sm, sm + DA * lda, colbuf, s_bad, d, x, x_next, status);
  }
}

template <int NBLK, bool INV>
cudaError_t launch_gram_ols_t(const double *SA, int64_t m, int d, double scale, const double *g, const double *x,
                              double *x_next, double *H_out, int *status, double *Hinv, int max_cluster,
                              cudaStream_t st) {
  constexpr int D = 32 * NBLK;
  const size_t smem_chol = ((size_t)(D + 8) * (D + 4) + D + (INV ? (size_t)NBLK * 32 * 36 : 0)) * 8;
  const size_t smem_gram = ((size_t)kGoRows * (D + 4) + (size_t)D * D) * 8;
  const size_t smem = std::max(smem_chol, smem_gram);
  auto kern = gram_ols_kernel<NBLK, INV>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaError_t e = cudaErrorUnknown;
  for (int cs : {16, 8, 4}) {
    if (cs > max_cluster) continue;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(kBThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, kern, SA, m, d, scale * scale, g, x, x_next, H_out, status, Hinv);
    if (e == cudaSuccess) return e;
    cudaGetLastError();
  }
  return e;
}

template <int NBLK>
void launch_blocked(const double *H, const double *g, int d, const double *x, double *x_next, int *status,
                    const int *run, cudaStream_t st) {
  constexpr int D = 32 * NBLK;
  const size_t smem = std::max(((size_t)(D + 8) * (D + 4) + D) * 8, kExclusiveSmem);
  IHS_SMEM_ATTR((chol_blocked_kernel<NBLK>), smem);
  chol_blocked_kernel<NBLK><<<1, kBThreads, smem, st>>>(H, g, d, x, x_next, status, run);
}
}  // namespace

size_t chol_scratch_bytes(int64_t d) { return d > 160 ? ols_large_scratch_bytes(d) : 256; }

bool gram_ols_supported(int64_t d) { return d >= 1 && d <= 128; }

cudaError_t launch_gram_ols(const double *SA, int64_t m, int64_t d, double scale, const double *g, const double *x,
                            double *x_next, double *H_out, int *status, cudaStream_t st, LaunchCounter lc) {
  cudaError_t e;
#define GO(NB) launch_gram_ols_t<NB, false>(SA, m, (int)d, scale, g, x, x_next, H_out, status, nullptr, 16, st)
  switch ((d + 31) / 32) {
    case 1: e = GO(1); break;
    case 2: e = GO(2); break;
    case 3: e = GO(3); break;
    default: e = GO(4); break;
  }
#undef GO
  lc.add();
  return e;
}

// The look-ahead factor: Hinv = (scale^2 SA^T SA)^{-1} in one cluster launch of
// at most max_cluster CTAs (it runs beside the sketch gather of the next pass,
// so it should leave that kernel's wave of bucket CTAs room on the other SMs).
cudaError_t launch_ols_factor(const double *SA, int64_t m, int64_t d, double scale, double *Hinv, int *status,
                              int max_cluster, cudaStream_t st, LaunchCounter lc) {
  cudaError_t e;
#define GO(NB) launch_gram_ols_t<NB, true>(SA, m, (int)d, scale, nullptr, nullptr, nullptr, nullptr, status, Hinv, \
                                           max_cluster, st)
  switch ((d + 31) / 32) {
    case 1: e = GO(1); break;
    case 2: e = GO(2); break;
    case 3: e = GO(3); break;
    default: e = GO(4); break;
  }
#undef GO
  lc.add();
  return e;
}

// x_next = x + Hinv g: one CTA, warp w owns rows w, w + 32, ...; lanes stride
// the row (coalesced) and a fixed shuffle tree sums them (deterministic).
__global__ void __launch_bounds__(1024) ols_apply_kernel(const double *__restrict__ Hinv,
                                                         const double *__restrict__ g, int d,
                                                         const double *__restrict__ x, double *x_next) {
  __shared__ double gs[1024];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int c = threadIdx.x; c < d; c += 1024) gs[c] = g[c];
  __syncthreads();
  // warp w rows 4w.., 4 rows x 4 column chunks of loads in flight before the adds
  const int nk = (d + 31) / 32;
  for (int i0 = warp * 4; i0 < d; i0 += 128) {
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int kb = 0; kb < nk; kb += 4) {
      double h[4][4];
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int c = lane + 32 * (kb + k);
          h[q][k] = (i0 + q < d && c < d) ? Hinv[(int64_t)(i0 + q) * d + c] * gs[c] : 0.0;
        }
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] += (h[q][0] + h[q][1]) + (h[q][2] + h[q][3]);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      double v = acc[q];
#pragma unroll
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0 && i0 + q < d) x_next[i0 + q] = x[i0 + q] + v;
    }
  }
}

cudaError_t launch_ols_apply(const double *Hinv, const double *g, int64_t d, const double *x, double *x_next,
                             cudaStream_t st, LaunchCounter lc) {
  if (d > 1024) return cudaErrorInvalidValue;
  ols_apply_kernel<<<1, 1024, 0, st>>>(Hinv, g, (int)d, x, x_next);
  lc.add();
  return cudaGetLastError();
}

cudaError_t launch_ols_update(const double *H, const double *g, int64_t d, const double *x, double *x_next,
                              double *scratch, int *status, int num_sms, int large_mode, cudaStream_t st,
                              LaunchCounter lc) {
  if (d <= 160) {
    const int *run = nullptr;
    const int nblk = (int)((d + 31) / 32);
    switch (nblk) {
      case 1: launch_blocked<1>(H, g, (int)d, x, x_next, status, run, st); break;
      case 2: launch_blocked<2>(H, g, (int)d, x, x_next, status, run, st); break;
      case 3: launch_blocked<3>(H, g, (int)d, x, x_next, status, run, st); break;
      case 4: launch_blocked<4>(H, g, (int)d, x, x_next, status, run, st); break;
      default: launch_blocked<5>(H, g, (int)d, x, x_next, status, run, st); break;
    }
    lc.add();
    return cudaGetLastError();
  }
  // d > 160: conjugate gradients with the blocked Cholesky behind them in the
  // same launch (ols_large.cu; large_mode 1), CG alone (0) or the Cholesky alone (2)
  if (!ols_large_supported(d)) return cudaErrorInvalidValue;
  return launch_ols_large(H, g, d, x, x_next, scratch, status, num_sms, large_mode, st, lc);
}

}  // namespace ihs
