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

template <int NV, int U, int W>
__global__ void __launch_bounds__(W * 32) grad_dense_kernel(const double *__restrict__ A, int64_t n, int d,
                                                                 const double *__restrict__ bvec,
                                                                 const double *__restrict__ x,
                                                                 double *__restrict__ gpart, int64_t rows_per_warp) {
  extern __shared__ double red[];  // W x d
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * W + warp;
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
    for (int w = 0; w < W; ++w) s += red[w * d + c];
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

// out[y*d + c] = sum over rows r in [y*rpb, min(rows, (y+1)*rpb)) of part[r*d + c]:
// blockIdx.y splits the rows, warp w sums rows r0+w, r0+w+W, ... ascending;
// then warp 0 adds the W warp sums in order.  Fixed order => deterministic.
__global__ void __launch_bounds__(1024) reduce_rows_kernel(const double *__restrict__ part, int64_t rows, int d,
                                                           int64_t rpb, double *__restrict__ out) {
  __shared__ double sm[32][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int c = blockIdx.x * 32 + lane;
  const int64_t r0 = (int64_t)blockIdx.y * rpb, r1 = min(rows, r0 + rpb);
  // 4 interleaved partial sums per thread (independent L2 loads in flight),
  // combined in a fixed order: deterministic
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  if (c < d) {
    int64_t r = r0 + warp;
    for (; r + 3 * nw < r1; r += 4 * nw) {
      s0 += part[r * d + c];
      s1 += part[(r + nw) * d + c];
      s2 += part[(r + 2 * nw) * d + c];
      s3 += part[(r + 3 * nw) * d + c];
    }
    for (; r < r1; r += nw) s0 += part[r * d + c];
  }
  const double s = (s0 + s1) + (s2 + s3);
  sm[warp][lane] = s;
  __syncthreads();
  if (warp == 0 && c < d) {
    double t = 0.0;
    for (int w = 0; w < nw; ++w) t += sm[w][lane];
    out[(int64_t)blockIdx.y * d + c] = t;
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

template <int NV, int U, int W = kWarps>
void launch_grad_t(const double *A, int64_t n, int d, const double *bvec, const double *x, double *gpart,
                   int64_t nblocks, cudaStream_t st) {
  const int64_t warps = nblocks * W;
  int64_t rpw = (n + warps - 1) / warps;
  rpw = (rpw + U - 1) / U * U;
  size_t smem = (size_t)W * d * 8;
  IHS_SMEM_ATTR((grad_dense_kernel<NV, U, W>), smem);
  grad_dense_kernel<NV, U, W><<<(unsigned)nblocks, W * 32, smem, st>>>(A, n, d, bvec, x, gpart, rpw);
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

int64_t reduce_rows_tmp(int64_t rows, int64_t d) {
  return ((rows + kReduceRowsPerCta - 1) / kReduceRowsPerCta) * d;
}

// One launch for out[c] = sum_r part[r*d + c]: CTA (x, y) sums rows
// [y*64, (y+1)*64) of columns [32x, 32x + 32) into tmp[y*d + c] (16 warps, a
// fixed order); the last CTA to finish (device-scope counter, left at 0) adds
// the R = gridDim.y partials of every column in order into out (deterministic)
// and, when Hinv is given, applies x_next = x + Hinv out (the look-ahead OLS
// step when no all-reduce separates the two, api.cu).  Replaces a d/32-CTA
// single level (9.9 us for 1024 x 128 on B200) and a second launch.
constexpr int kRedThreads = 512;
__global__ void __launch_bounds__(kRedThreads) reduce_rows_last_kernel(
    const double *__restrict__ part, int64_t rows, int d, double *tmp, double *out, unsigned *counter,
    const double *__restrict__ Hinv, const double *__restrict__ x, double *x_next) {
  constexpr int NW = kRedThreads / 32;
  __shared__ double sm[NW][33];
  __shared__ double gs[1024];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane;
  const int64_t r0 = (int64_t)blockIdx.y * kReduceRowsPerCta, r1 = min(rows, r0 + kReduceRowsPerCta);
  static_assert(kReduceRowsPerCta == 4 * NW, "four rows per warp");
  // rows r0 + warp + NW k (k < 4 covers the 64 rows): loads first, then the adds
  // in k order, so the four L2 round trips overlap (a runtime-bounded loop
  // would issue each load only after the previous add)
  double v[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int64_t r = r0 + warp + NW * k;
    v[k] = (c < d && r < r1) ? part[r * d + c] : 0.0;
  }
  sm[warp][lane] = (v[0] + v[1]) + (v[2] + v[3]);
  __syncthreads();
  if (warp == 0 && c < d) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) t += sm[w][lane];
    tmp[(int64_t)blockIdx.y * d + c] = t;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x * gridDim.y - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  const int R = gridDim.y;
  for (int cc = threadIdx.x; cc < d; cc += kRedThreads) {
    double acc = 0.0;
    for (int y0 = 0; y0 < R; y0 += 8) {  // 8 loads in flight, added in y order
      double u[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) u[k] = (y0 + k < R) ? __ldcg(tmp + (int64_t)(y0 + k) * d + cc) : 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) acc += u[k];
    }
    out[cc] = acc;
    gs[cc] = acc;
  }
  if (threadIdx.x == 0) *counter = 0;
  if (!Hinv) return;
  __syncthreads();
  // x_next = x + Hinv g: warp w rows 4w.., 4 rows x 4 column chunks of loads in flight
  const int nk = (d + 31) / 32;
  for (int i0 = warp * 4; i0 < d; i0 += NW * 4) {
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int kb = 0; kb < nk; kb += 4) {
      double h[4][4];
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int cc = lane + 32 * (kb + k);
          h[q][k] = (i0 + q < d && cc < d) ? __ldcg(Hinv + (int64_t)(i0 + q) * d + cc) * gs[cc] : 0.0;
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

cudaError_t launch_reduce_rows(const double *part, int64_t rows, int64_t d, double *out, double *tmp,
                               unsigned *counter, cudaStream_t st, LaunchCounter lc, const double *Hinv,
                               const double *x, double *x_next) {
  if (d > 1024) return cudaErrorInvalidValue;
  const unsigned gx = (unsigned)((d + 31) / 32);
  const int64_t R = std::max<int64_t>(1, (rows + kReduceRowsPerCta - 1) / kReduceRowsPerCta);
  if (R > 65535) {  // (> 4M partial rows) one level over d/32 CTAs, then the update apart
    reduce_rows_kernel<<<gx, 1024, 0, st>>>(part, rows, (int)d, rows, out);
    lc.add();
    if (Hinv) return launch_ols_apply(Hinv, out, d, x, x_next, st, lc);
    return cudaGetLastError();
  }
  reduce_rows_last_kernel<<<dim3(gx, (unsigned)R), kRedThreads, 0, st>>>(part, rows, (int)d, tmp, out, counter,
                                                                          Hinv, x, x_next);
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
    reduce_rows_kernel<<<1, 1024, 0, st>>>(part, nblocks, 1, nblocks, err2 + k);
    lc.add(3);
  }
  return cudaGetLastError();
}

}  // namespace ihs
