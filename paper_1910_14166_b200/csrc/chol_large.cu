// a6, OLS for large d (d > 160, e.g. BASELINE.json configs[2], d = 1024):
// blocked right-looking Cholesky across the GPU in 64-column panels, on an
// augmented matrix [[H, g], [g^T, *]] so that row d of the factor is the
// forward-substitution result y = L^{-1} g for free.  Per panel kb:
//   potrf  (1 CTA)   factor the 64x64 diagonal block in shared memory;
//   trsm   (n CTAs)  rows below solve X L11^T = A21, one thread per row;
//   syrk   (n CTAs)  trailing lower 64x64 tiles -= L21 L21^T on the DMMA pipe.
// Then one CTA runs the blocked back substitution L^T u = y and x + u.
// Eq. (2) with C = R^d; T_solve = O(d^3).
#include "common.cuh"
#include "kernels.h"
#include "chol_blocks.cuh"

namespace ihs {

namespace {
constexpr int PB = 64;         // panel width
constexpr int LDP = PB + 4;    // smem row stride (== 4 mod 16 doubles)

__device__ __forceinline__ void dmma884(double &c0, double &c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__global__ void aug_fill_kernel(const double *__restrict__ H, const double *__restrict__ g, int d, int Dp,
                                double *__restrict__ M, int *flag) {
  const int64_t total = (int64_t)Dp * Dp;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / Dp), c = (int)(e % Dp);
    double v = 0.0;
    if (c <= i) {
      if (i < d) v = H[(int64_t)i * d + c];
      else if (i == d) v = c < d ? g[c] : 1.0;
      else v = (c == i) ? 1.0 : 0.0;
    }
    M[e] = v;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *flag = 0;
}

// Factor the diagonal 64x64 block at (kb, kb) in shared memory.
__global__ void __launch_bounds__(256) potrf_diag_kernel(double *__restrict__ M, int Dp, int kb, int d,
                                                         double *__restrict__ rdiag, int *flag, int *status) {
  __shared__ double Ls[PB * LDP];
  __shared__ double rd[PB];
  __shared__ int s_bad;
  __shared__ double colbuf[64];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (*flag) return;  // an earlier panel failed: nothing left to do
  for (int i = warp; i < PB; i += 8)
    for (int c = lane; c <= i; c += 32) Ls[i * LDP + c] = M[(int64_t)(kb + i) * Dp + kb + c];
  if (tid == 0) s_bad = 0;
  __syncthreads();
  for (int k2 = 0; k2 < PB; k2 += 32) {
    if (warp == 0) {
      const bool bad = warp_chol32(Ls + k2 * LDP + k2, LDP, rd + k2, d - (kb + k2), colbuf);
      if (bad && lane == 0) s_bad = 1;
    }
    __syncthreads();
    if (s_bad) break;
    if (k2 == 0) {
      if (tid < 32) thread_trsm32(Ls + (32 + tid) * LDP, Ls, LDP, rd);  // rows 32..63 against the first block
      __syncthreads();
      // lower 8x8 tiles of the (32,32) block -= L21 L21^T
      for (int t = warp; t < 10; t += 8) {
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
        const int r = I + (lane >> 2), c = J + 2 * (lane & 3);
        Ls[r * LDP + c] -= c0;
        Ls[r * LDP + c + 1] -= c1;
      }
      __syncthreads();
    }
  }
  if (s_bad) {
    if (tid == 0) {
      *flag = 1;
      set_status(status, 3 /* IHS_ERR_NOT_SPD */);
    }
    return;
  }
  for (int i = warp; i < PB; i += 8)
    for (int c = lane; c <= i; c += 32) M[(int64_t)(kb + i) * Dp + kb + c] = Ls[i * LDP + c];
  if (tid < PB) rdiag[kb + tid] = rd[tid];
}

// Rows below the panel: X L11^T = A21, one thread per row.  With L11 =
// [[P, 0], [Q, R]] (32x32 blocks): x1 P^T = a1, then x2 R^T = a2 - x1 Q^T.
// Each thread stages its 64-wide row in shared memory (stride 65: conflict-free
// across threads); L11 is read as broadcasts.
constexpr int kTrsmThreads = 128;
__global__ void __launch_bounds__(kTrsmThreads) trsm_panel_kernel(double *__restrict__ M, int Dp, int kb,
                                                                  const double *__restrict__ rdiag, const int *flag) {
  extern __shared__ double tsm[];
  double *L11 = tsm;                  // PB x (PB + 1)
  double *X = L11 + PB * (PB + 1);    // kTrsmThreads x (PB + 1)
  double *rd = X + kTrsmThreads * (PB + 1);
  if (*flag) return;
  for (int e = threadIdx.x; e < PB * PB; e += blockDim.x) {
    const int i = e / PB, c = e % PB;
    L11[i * (PB + 1) + c] = (c <= i) ? M[(int64_t)(kb + i) * Dp + kb + c] : 0.0;
  }
  if (threadIdx.x < PB) rd[threadIdx.x] = rdiag[kb + threadIdx.x];
  const int r0 = kb + PB + blockIdx.x * blockDim.x;
  const int nr = min((int)blockDim.x, Dp - r0);
  for (int e = threadIdx.x; e < nr * PB; e += blockDim.x) {  // coalesced: consecutive threads, consecutive columns
    const int r = e / PB, c = e % PB;
    X[r * (PB + 1) + c] = M[(int64_t)(r0 + r) * Dp + kb + c];
  }
  __syncthreads();
  double *x = X + threadIdx.x * (PB + 1);
  if (threadIdx.x < nr) {
    thread_trsm32(x, L11, PB + 1, rd);
    const double *Q = L11 + 32 * (PB + 1);
#pragma unroll 1
    for (int c = 0; c < 32; ++c) {
      double t0 = 0.0, t1 = 0.0;
#pragma unroll
      for (int k = 0; k < 32; k += 2) {
        t0 = fma(x[k], Q[c * (PB + 1) + k], t0);
        t1 = fma(x[k + 1], Q[c * (PB + 1) + k + 1], t1);
      }
      x[32 + c] -= t0 + t1;
    }
    thread_trsm32(x + 32, L11 + 32 * (PB + 1) + 32, PB + 1, rd + 32);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nr * PB; e += blockDim.x) {
    const int r = e / PB, c = e % PB;
    M[(int64_t)(r0 + r) * Dp + kb + c] = X[r * (PB + 1) + c];
  }
}

// Trailing update of the lower 64x64 tiles: C_IJ -= P_I P_J^T with P = the
// panel's 64 columns (DMMA, 4 warps x 32x32 sub-tiles).
__global__ void __launch_bounds__(128) syrk_panel_kernel(double *__restrict__ M, int Dp, int kb, const int *flag) {
  extern __shared__ double sm[];
  double *PI = sm;              // [k][r], PB x LDP
  double *PJ = sm + PB * LDP;   // [k][r]
  if (*flag) return;
  const int t0 = kb + PB;
  int ti = 0, rem = blockIdx.x;  // lower tiles, row-major
  while (rem > ti) {
    rem -= ti + 1;
    ++ti;
  }
  const int I = t0 + PB * ti, J = t0 + PB * rem;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < PB * PB; e += blockDim.x) {
    const int r = e / PB, k = e % PB;
    PI[k * LDP + r] = M[(int64_t)(I + r) * Dp + kb + k];
    PJ[k * LDP + r] = M[(int64_t)(J + r) * Dp + kb + k];
  }
  __syncthreads();
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
      const int c = J + 32 * wn + 8 * b + 2 * (lane & 3);
      double *p = M + (int64_t)r * Dp + c;
      p[0] -= acc[a][b][0];
      p[1] -= acc[a][b][1];
    }
}

// Back substitution L^T u = y (y = row d of the augmented factor), then
// x_next = x + u; x_next = x when a pivot failed.
__global__ void __launch_bounds__(1024) backsolve_kernel(const double *__restrict__ M, int Dp, int d,
                                                         const double *__restrict__ rdiag,
                                                         const double *__restrict__ x, double *x_next,
                                                         const int *flag) {
  extern __shared__ double sm[];
  double *z = sm;               // d
  double *Lp = sm + d;          // PB x (PB + 1)
  const int tid = threadIdx.x, lane = tid & 31;
  if (*flag) {
    for (int k = tid; k < d; k += blockDim.x) x_next[k] = x[k];
    return;
  }
  for (int k = tid; k < d; k += blockDim.x) z[k] = M[(int64_t)d * Dp + k];
  __syncthreads();
  for (int kb = ((d - 1) / PB) * PB; kb >= 0; kb -= PB) {
    const int w = min(PB, d - kb);
    for (int e = tid; e < PB * PB; e += blockDim.x) {
      const int i = e / PB, c = e % PB;
      Lp[i * (PB + 1) + c] = (i < w && c <= i) ? M[(int64_t)(kb + i) * Dp + kb + c] : 0.0;
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
          const double ui = __shfl_sync(0xffffffffu, zr[s], jj) * rdiag[kb + i];
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
    // z[k] -= sum_i L[kb+i][k] u[kb+i] for k < kb: coalesced rows of L from L2,
    // 16 independent loads in flight per thread (rows >= w of the block are the
    // identity padding / zero and never read: w == PB except for the top block)
    for (int k = tid; k < kb; k += blockDim.x) {
      const double *col = M + (int64_t)kb * Dp + k;
      double t0 = 0.0, t1 = 0.0;
      if (w == PB) {
#pragma unroll 16
        for (int i = 0; i < PB; i += 2) {
          t0 = fma(col[(int64_t)i * Dp], z[kb + i], t0);
          t1 = fma(col[(int64_t)(i + 1) * Dp], z[kb + i + 1], t1);
        }
      } else {
        for (int i = 0; i < w; ++i) t0 = fma(col[(int64_t)i * Dp], z[kb + i], t0);
      }
      z[k] -= t0 + t1;
    }
    __syncthreads();
  }
  for (int k = tid; k < d; k += blockDim.x) x_next[k] = x[k] + z[k];
}
}  // namespace

size_t chol_large_scratch_bytes(int64_t d) {
  const int64_t Dp = (d + 1 + PB - 1) / PB * PB;
  return (size_t)(Dp * Dp + Dp) * 8 + 64;
}

cudaError_t launch_chol_large(const double *H, const double *g, int64_t d, const double *x, double *x_next,
                              double *scratch, int *status, cudaStream_t st, LaunchCounter lc) {
  const int Dp = (int)((d + 1 + PB - 1) / PB * PB);
  double *M = scratch;
  double *rdiag = scratch + (size_t)Dp * Dp;
  int *flag = reinterpret_cast<int *>(rdiag + Dp);
  const int64_t total = (int64_t)Dp * Dp;
  aug_fill_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, 148 * 8), 256, 0, st>>>(H, g, (int)d, Dp, M,
                                                                                             flag);
  int launches = 1;
  const size_t syrk_smem = (size_t)2 * PB * LDP * 8;
  IHS_SMEM_ATTR(syrk_panel_kernel, syrk_smem);
  const size_t trsm_smem = ((size_t)(PB + kTrsmThreads) * (PB + 1) + PB) * 8;
  IHS_SMEM_ATTR(trsm_panel_kernel, trsm_smem);
  for (int kb = 0; kb < Dp; kb += PB) {
    potrf_diag_kernel<<<1, 256, 0, st>>>(M, Dp, kb, (int)d, rdiag, flag, status);
    const int below = Dp - kb - PB;
    ++launches;
    if (below > 0) {
      trsm_panel_kernel<<<(below + kTrsmThreads - 1) / kTrsmThreads, kTrsmThreads, trsm_smem, st>>>(M, Dp, kb, rdiag, flag);
      const int nt = below / PB;
      syrk_panel_kernel<<<nt * (nt + 1) / 2, 128, syrk_smem, st>>>(M, Dp, kb, flag);
      launches += 2;
    }
  }
  const size_t bs_smem = ((size_t)d + PB * (PB + 1)) * 8;
  IHS_SMEM_ATTR(backsolve_kernel, bs_smem);
  backsolve_kernel<<<1, 1024, bs_smem, st>>>(M, Dp, (int)d, rdiag, x, x_next, flag);
  lc.add(launches + 1);
  return cudaGetLastError();
}

}  // namespace ihs
