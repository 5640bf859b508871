// a5: g = A^T (b - A x) for dense row-major A in one pass (Eq. (2) linear term,
// PAPER.md:83-86; "any further access to A is for matrix-vector products",
// PAPER.md:95-96), plus the fixed-order partial reductions and the a7 error
// norm ||A v||^2.  HBM-bound streaming kernels: each warp reads U whole rows
// per step with coalesced loads, transpose-reduces the U dot products, and
// accumulates r_i a_i in registers.  Deterministic (fixed reduction order).
#include "common.cuh"
#include "kernels.h"

namespace ihs {

namespace {
constexpr int kWarps = 8;

template <int NV, int U>
__global__ void __launch_bounds__(kWarps * 32) grad_dense_kernel(const double *__restrict__ A, int64_t n, int d,
                                                                 const double *__restrict__ bvec,
                                                                 const double *__restrict__ x,
                                                                 double *__restrict__ gpart, int64_t rows_per_warp) {
  extern __shared__ double red[];  // kWarps x d
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * kWarps + warp;
  const int64_t r0 = min(n, gw * rows_per_warp);
  const int64_t r1 = min(n, r0 + rows_per_warp);
  // unpredicated loads from clamped addresses (see cs_gather.cu); clamped
  // columns carry x = 0 and clamped rows carry r = 0.
  int col[NV], colc[NV];
  bool cval[NV];
  double xv[NV], gacc[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    col[k] = lane + 32 * k;
    cval[k] = col[k] < d;
    colc[k] = cval[k] ? col[k] : d - 1;
    xv[k] = cval[k] ? x[col[k]] : 0.0;
    gacc[k] = 0.0;
  }
#pragma unroll 1
  for (int64_t base = r0; base < r1; base += U) {
    double v[U][NV];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t row = (base + u < r1) ? base + u : r1 - 1;
      const double *rowp = A + row * d;
#pragma unroll
      for (int k = 0; k < NV; ++k) v[u][k] = ldg_stream(rowp + colc[k]);
    }
    double p[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      p[u] = 0.0;
#pragma unroll
      for (int k = 0; k < NV; ++k) p[u] = fma(v[u][k], xv[k], p[u]);
    }
    transpose_reduce<U>(p, lane);
    const int myu = reduced_row_of_lane<U>(lane);
    const double res = (base + myu < r1) ? bvec[base + myu] - p[0] : 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const double ru = __shfl_sync(0xffffffffu, res, owner_lane_of_row<U>(u));
#pragma unroll
      for (int k = 0; k < NV; ++k) gacc[k] = fma(ru, v[u][k], gacc[k]);
    }
  }
#pragma unroll
  for (int k = 0; k < NV; ++k)
    if (cval[k]) red[warp * d + col[k]] = gacc[k];
  __syncthreads();
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) s += red[w * d + c];
    gpart[(int64_t)blockIdx.x * d + c] = s;
  }
}

// ||A v||^2 partial per CTA (a7 error norm).
template <int NV, int U>
__global__ void __launch_bounds__(kWarps * 32) sqnorm_dense_kernel(const double *__restrict__ A, int64_t n, int d,
                                                                   const double *__restrict__ vvec,
                                                                   double *__restrict__ part, int64_t rows_per_warp) {
  __shared__ double red[kWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * kWarps + warp;
  const int64_t r0 = min(n, gw * rows_per_warp);
  const int64_t r1 = min(n, r0 + rows_per_warp);
  double xv[NV];
  int colc[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const int c = lane + 32 * k;
    colc[k] = c < d ? c : d - 1;
    xv[k] = c < d ? vvec[c] : 0.0;
  }
  double acc = 0.0;
  const int myu = reduced_row_of_lane<U>(lane);
  const bool owner = owner_lane_of_row<U>(myu) == lane;
#pragma unroll 1
  for (int64_t base = r0; base < r1; base += U) {
    double p[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t row = (base + u < r1) ? base + u : r1 - 1;
      const double *rowp = A + row * d;
      p[u] = 0.0;
#pragma unroll
      for (int k = 0; k < NV; ++k) p[u] = fma(ldg_stream(rowp + colc[k]), xv[k], p[u]);
    }
    transpose_reduce<U>(p, lane);
    if (owner && base + myu < r1) acc = fma(p[0], p[0], acc);
  }
  acc = warp_sum(acc);
  if (lane == 0) red[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kWarps; ++w) s += red[w];
    part[blockIdx.x] = s;
  }
}

__global__ void sqnorm_csr_kernel(int64_t n, const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                                  const double *__restrict__ val, const double *__restrict__ vvec,
                                  double *__restrict__ part) {
  __shared__ double red[32];
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double dot = 0.0;
    for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) dot = fma(val[e], vvec[col[e]], dot);
    acc = fma(dot, dot, acc);
  }
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    part[blockIdx.x] = s;
  }
}

// out[c] = sum_r part[r*d + c]: warp w sums rows w, w+32, ... ascending; then
// warp 0 adds the 32 warp sums in order.  Fixed order => deterministic.
__global__ void __launch_bounds__(1024) reduce_rows_kernel(const double *__restrict__ part, int64_t rows, int d,
                                                           double *__restrict__ out) {
  __shared__ double sm[32][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane;
  // 4 interleaved partial sums per thread (independent L2 loads in flight),
  // combined in a fixed order: deterministic
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  if (c < d) {
    int64_t r = warp;
    for (; r + 96 < rows; r += 128) {
      s0 += part[r * d + c];
      s1 += part[(r + 32) * d + c];
      s2 += part[(r + 64) * d + c];
      s3 += part[(r + 96) * d + c];
    }
    for (; r < rows; r += 32) s0 += part[r * d + c];
  }
  const double s = (s0 + s1) + (s2 + s3);
  sm[warp][lane] = s;
  __syncthreads();
  if (warp == 0 && c < d) {
    double t = 0.0;
    for (int w = 0; w < 32; ++w) t += sm[w][lane];
    out[c] = t;
  }
}

__global__ void scale_kernel(double *__restrict__ buf, int64_t count, double scale) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    buf[i] = buf[i] * scale;
}

__global__ void axpy_diff_kernel(const double *__restrict__ a, const double *__restrict__ b, int d, double *out) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < d) out[c] = b ? a[c] - b[c] : a[c];
}

template <int NV, int U>
void launch_grad_t(const double *A, int64_t n, int d, const double *bvec, const double *x, double *gpart,
                   int64_t nblocks, cudaStream_t st) {
  const int64_t warps = nblocks * kWarps;
  int64_t rpw = (n + warps - 1) / warps;
  rpw = (rpw + U - 1) / U * U;
  size_t smem = (size_t)kWarps * d * 8;
  IHS_SMEM_ATTR((grad_dense_kernel<NV, U>), smem);
  grad_dense_kernel<NV, U><<<(unsigned)nblocks, kWarps * 32, smem, st>>>(A, n, d, bvec, x, gpart, rpw);
}

template <int NV, int U>
void launch_sqnorm_t(const double *A, int64_t n, int d, const double *v, double *part, int64_t nblocks,
                     cudaStream_t st) {
  const int64_t warps = nblocks * kWarps;
  int64_t rpw = (n + warps - 1) / warps;
  rpw = (rpw + U - 1) / U * U;
  sqnorm_dense_kernel<NV, U><<<(unsigned)nblocks, kWarps * 32, 0, st>>>(A, n, d, v, part, rpw);
}
}  // namespace

int64_t grad_dense_blocks(int64_t n, int64_t d, int num_sms) {
  (void)d;
  int64_t want = (int64_t)num_sms * 4;
  int64_t maxb = std::max<int64_t>(1, (n + 31) / 32);
  return std::max<int64_t>(1, std::min(want, maxb));
}

#define IHS_NV_DISPATCH(nv, CALL)            \
  switch (nv) {                              \
    case 1: CALL(1, 16); break;              \
    case 2: CALL(2, 16); break;              \
    case 3: CALL(3, 8); break;               \
    case 4: CALL(4, 8); break;               \
    case 5:                                  \
    case 6: CALL(6, 4); break;               \
    case 7:                                  \
    case 8: CALL(8, 4); break;               \
    case 9: case 10: case 11: case 12:       \
    case 13: case 14: case 15: case 16:      \
      CALL(16, 2); break;                    \
    default: CALL(32, 1); break;             \
  }

cudaError_t launch_grad_dense(const double *A, int64_t n, int64_t d, const double *bvec, const double *x,
                              double *gpart, int64_t nblocks, cudaStream_t st, LaunchCounter lc) {
  if (d > 1024) return cudaErrorInvalidValue;
  const int nv = (int)((d + 31) / 32);
#define CALL(NV, U) launch_grad_t<NV, U>(A, n, (int)d, bvec, x, gpart, nblocks, st)
  IHS_NV_DISPATCH(nv, CALL)
#undef CALL
  lc.add();
  return cudaGetLastError();
}

cudaError_t launch_reduce_rows(const double *part, int64_t rows, int64_t d, double *out, cudaStream_t st,
                               LaunchCounter lc) {
  reduce_rows_kernel<<<(unsigned)((d + 31) / 32), 1024, 0, st>>>(part, rows, (int)d, out);
  lc.add();
  return cudaGetLastError();
}

cudaError_t launch_scale(double *buf, int64_t count, double scale, cudaStream_t st, LaunchCounter lc) {
  if (count <= 0) return cudaSuccess;
  int grid = (int)std::min<int64_t>((count + 255) / 256, 148 * 8);
  scale_kernel<<<grid, 256, 0, st>>>(buf, count, scale);
  lc.add();
  return cudaGetLastError();
}

// err2[k] = ||A (X[k] - xref)||^2 for k < count, err2[count] = ||A xref||^2.
// scratch: d + nblocks doubles.
cudaError_t launch_pred_err2_impl(int layout, int64_t n, int64_t d, const double *values, const int64_t *row_ptr,
                                  const int32_t *col, const double *X, int count, const double *xref,
                                  double *err2, double *scratch, int num_sms, cudaStream_t st, LaunchCounter lc) {
  if (layout == 0 && d > 1024) return cudaErrorInvalidValue;
  double *v = scratch;
  double *part = scratch + ((d + 31) / 32) * 32;
  const int64_t nblocks = grad_dense_blocks(n, d, num_sms);
  const int nv = (int)((d + 31) / 32);
  for (int k = 0; k <= count; ++k) {
    axpy_diff_kernel<<<(unsigned)((d + 127) / 128), 128, 0, st>>>(k < count ? X + (int64_t)k * d : xref,
                                                                    k < count ? xref : nullptr, (int)d, v);
    if (layout == 0) {
#define CALL(NV, U) launch_sqnorm_t<NV, U>(values, n, (int)d, v, part, nblocks, st)
      IHS_NV_DISPATCH(nv, CALL)
#undef CALL
    } else {
      sqnorm_csr_kernel<<<(unsigned)nblocks, 256, 0, st>>>(n, row_ptr, col, values, v, part);
    }
    reduce_rows_kernel<<<1, 1024, 0, st>>>(part, nblocks, 1, err2 + k);
    lc.add(3);
  }
  return cudaGetLastError();
}

}  // namespace ihs
