// a6, OLS: x^{t+1} = x^t + H^{-1} g (Eq. (2) with C = R^d, PAPER.md:83-86;
// T_solve = O(d^3)).  Right-looking Cholesky H = L L^T in
// one CTA (H in shared memory when d^2 * 8 fits, else in an L2-resident global
// scratch), then forward / back substitution by one warp and the update
// x + u.  A pivot <= 0 sets IHS_ERR_NOT_SPD (reading R13) and x_next = x.
// Latency-bound: d = 10..256 take O(d) barrier steps.
#include "common.cuh"
#include "kernels.h"

namespace ihs {

namespace {
constexpr int kThreads = 512;
constexpr size_t kSmemLimit = 200 * 1024;

__global__ void __launch_bounds__(kThreads) chol_solve_kernel(const double *__restrict__ H,
                                                              const double *__restrict__ g, int d,
                                                              const double *__restrict__ x, double *x_next,
                                                              double *scratch, int *status, int use_smem) {
  extern __shared__ double sm[];
  double *a = use_smem ? sm : scratch;  // d x d, lower triangle overwritten by L
  double *z = use_smem ? sm + (size_t)d * d : scratch + (size_t)d * d;  // d
  __shared__ double s_ljj;
  __shared__ int s_bad;
  const int tid = threadIdx.x;
  for (int64_t e = tid; e < (int64_t)d * d; e += blockDim.x) a[e] = H[e];
  for (int i = tid; i < d; i += blockDim.x) z[i] = g[i];
  if (tid == 0) s_bad = 0;
  __syncthreads();
  for (int j = 0; j < d; ++j) {
    if (tid == 0) {
      double piv = a[(int64_t)j * d + j];
      if (!(piv > 0.0)) {
        s_bad = 1;
      } else {
        double l = sqrt(piv);
        a[(int64_t)j * d + j] = l;
        s_ljj = l;
      }
    }
    __syncthreads();
    if (s_bad) break;
    const double ljj = s_ljj;
    for (int i = j + 1 + tid; i < d; i += blockDim.x) a[(int64_t)i * d + j] /= ljj;
    __syncthreads();
    // trailing update of the lower triangle: a[i][k] -= L[i][j] L[k][j], j < k <= i
    const int w = d - j - 1;
    for (int64_t idx = tid; idx < (int64_t)w * w; idx += blockDim.x) {
      int i = j + 1 + (int)(idx / w);
      int k = j + 1 + (int)(idx % w);
      if (k <= i) a[(int64_t)i * d + k] -= a[(int64_t)i * d + j] * a[(int64_t)k * d + j];
    }
    __syncthreads();
  }
  if (s_bad) {
    for (int i = tid; i < d; i += blockDim.x) x_next[i] = x[i];
    if (tid == 0) set_status(status, 3 /* IHS_ERR_NOT_SPD */);
    return;
  }
  if (tid < 32) {
    const int lane = tid;
    // forward: L y = g (column-oriented; row i subtracts terms j = 0..i-1 in order)
    for (int j = 0; j < d; ++j) {
      __syncwarp();
      const double yj = z[j] / a[(int64_t)j * d + j];
      __syncwarp();
      if (lane == 0) z[j] = yj;
      for (int i = j + 1 + lane; i < d; i += 32) z[i] -= a[(int64_t)i * d + j] * yj;
    }
    // backward: L^T u = y
    for (int i = d - 1; i >= 0; --i) {
      __syncwarp();
      const double ui = z[i] / a[(int64_t)i * d + i];
      __syncwarp();
      if (lane == 0) z[i] = ui;
      for (int k = lane; k < i; k += 32) z[k] -= a[(int64_t)i * d + k] * ui;
    }
    __syncwarp();
    for (int i = lane; i < d; i += 32) x_next[i] = x[i] + z[i];
  }
}
}  // namespace

size_t chol_scratch_bytes(int64_t d) { return (size_t)(d * d + d) * 8; }

cudaError_t launch_ols_update(const double *H, const double *g, int64_t d, const double *x, double *x_next,
                              double *scratch, int *status, int num_sms, cudaStream_t st, LaunchCounter lc) {
  (void)num_sms;
  const size_t need = (size_t)(d * d + d) * 8;
  const int use_smem = need <= kSmemLimit;
  const size_t smem = use_smem ? need : 0;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(chol_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  chol_solve_kernel<<<1, kThreads, smem, st>>>(H, g, (int)d, x, x_next, scratch, status, use_smem);
  lc.add();
  return cudaGetLastError();
}

}  // namespace ihs
