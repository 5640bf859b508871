// a2 + a5 for CSR A (BASELINE.json configs[2]): one streaming pass over the
// CSR arrays.  Each stored entry (i, c, v) is added into its s buckets
// (O(s nnz(A))), and r_i = b_i - a_i.x feeds g += r_i a_i
// (Eq. (2)).  With ~1 nonzero per row there is no reuse inside a row, so the
// sketch scatters with native fp64 reductions into an L2-resident SA
// (REDG.E.ADD.F64) and the gradient accumulates per CTA in shared memory
// before one flush.  The summation order is not fixed (documented tolerance,
// DESIGN.md section 6).
#include "common.cuh"
#include "kernels.h"

namespace ihs {

namespace {
// L2 eviction-priority policies: the CSR arrays and b stream through L2 once
// (evict_first); the reductions into SA keep its lines resident (evict_last),
// so the 34 M REDs of C3 do not re-fetch SA lines the stream pushed out.
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
template <typename T>
__device__ __forceinline__ T ld_stream(const T *p, uint64_t pol);
template <>
__device__ __forceinline__ double ld_stream<double>(const double *p, uint64_t pol) {
  double v;
  asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
template <>
__device__ __forceinline__ int32_t ld_stream<int32_t>(const int32_t *p, uint64_t pol) {
  int32_t v;
  asm volatile("ld.global.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
template <>
__device__ __forceinline__ int64_t ld_stream<int64_t>(const int64_t *p, uint64_t pol) {
  int64_t v;
  asm volatile("ld.global.L2::cache_hint.s64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void red_keep(double *p, double v, uint64_t pol) {
  asm volatile("red.global.add.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}

// Warp-compacted rows: a warp reads the row pointers of 128 consecutive rows
// (4 per lane), keeps the non-empty ones (~64% for C3's density) in a
// compacted order (ballots) and processes them 32 at a time, one row per
// lane.  The per-row work (s hashes, the dot product, s REDs per nonzero) then
// runs with nearly full warps; thread per row kept ~40% of the lanes active
// (ncu: 12.6 threads per warp instruction, issue-bound at 68% issue-active).
// Each lane's row loads (its first two nonzeros, b, x[col]) are issued before
// their first use.
constexpr int kRowsPerLane = 4;

// One row's work.  SC = s when it is known at compile time (1..8; 0: the
// runtime s).  The first two nonzeros (the common case at density 1e-3) are
// handled as predicated straight-line code; longer rows loop over the rest.
template <bool SKETCH, bool GRAD, bool GSMEM, int SC>
__device__ __forceinline__ void csr_row(int64_t i, int64_t e0, int64_t e1, int d, const int32_t *__restrict__ col,
                                        const double *__restrict__ val, int64_t row_offset, uint64_t key, uint32_t M,
                                        int s_rt, double scale, double *SA, const double *__restrict__ bvec,
                                        const double *__restrict__ x, double *g, double *gs, uint64_t pf,
                                        uint64_t pl) {
  const int s = SC > 0 ? SC : s_rt;
  const int nn = (int)(e1 - e0);
  const bool has1 = nn > 1;
  const int32_t c0 = ld_stream(col + e0, pf);
  const double v0 = ld_stream(val + e0, pf);
  const int32_t c1 = has1 ? ld_stream(col + e0 + 1, pf) : c0;
  const double v1 = has1 ? ld_stream(val + e0 + 1, pf) : 0.0;
  const double bi = GRAD ? ld_stream(bvec + i, pf) : 0.0;
  if (GRAD) {
    double dot = v0 * x[c0];
    if (has1) dot = fma(v1, x[c1], dot);
    for (int q = 2; q < nn; ++q) dot = fma(ld_stream(val + e0 + q, pf), x[ld_stream(col + e0 + q, pf)], dot);
    const double res = bi - dot;
    double *gt = GSMEM ? gs : g;
    atomicAdd(&gt[c0], v0 * res);
    if (has1) atomicAdd(&gt[c1], v1 * res);
    for (int q = 2; q < nn; ++q) atomicAdd(&gt[col[e0 + q]], val[e0 + q] * res);
  }
  if (SKETCH) {
    // S's entries are +-1/sqrt(s): the scale rides on each
    // reduced value (exact for s = 1, 4: a power of two) -- no pass over SA
    const double w0 = v0 * scale, w1 = v1 * scale;
#pragma unroll
    for (int j = 0; j < (SC > 0 ? SC : 1); ++j) {
      for (int jj = j; jj < s; jj += (SC > 0 ? SC : 1)) {  // SC > 0: exactly once
        bool neg;
        const uint32_t b = hash_bucket(key, (uint64_t)(row_offset + i), (uint32_t)jj, (uint32_t)s, M, neg);
        double *row = SA + (int64_t)b * d;
        red_keep(row + c0, neg ? -w0 : w0, pl);
        if (has1) red_keep(row + c1, neg ? -w1 : w1, pl);
        for (int q = 2; q < nn; ++q) {
          const double vq = val[e0 + q] * scale;
          red_keep(row + col[e0 + q], neg ? -vq : vq, pl);
        }
        if (SC > 0) break;
      }
    }
  }
}

template <bool SKETCH, bool GRAD, bool GSMEM, int SC>
__global__ void __launch_bounds__(256, 3) csr_sketch_grad_kernel(int64_t n, int d, const int64_t *__restrict__ row_ptr,
                                                                 const int32_t *__restrict__ col,
                                                                 const double *__restrict__ val, int64_t row_offset,
                                                                 uint64_t key, uint32_t M, int s, double scale,
                                                                 double *SA, const double *__restrict__ bvec,
                                                                 const double *__restrict__ x, double *g) {
  extern __shared__ double gs[];
  if (GRAD && GSMEM) {
    for (int c = threadIdx.x; c < d; c += blockDim.x) gs[c] = 0.0;
    __syncthreads();
  }
  const uint64_t pf = policy_evict_first(), pl = policy_evict_last();
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  __shared__ int64_t cbuf_e[2][8][32 * kRowsPerLane];  // per warp: compacted extents
  __shared__ int32_t cbuf_r[8][32 * kRowsPerLane];     // per warp: compacted rows (window offsets)
  int64_t *ce0 = cbuf_e[0][threadIdx.x >> 5], *ce1 = cbuf_e[1][threadIdx.x >> 5];
  int32_t *crow = cbuf_r[threadIdx.x >> 5];
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  constexpr int W = 32 * kRowsPerLane;
  for (int64_t base = warp * W; base < n; base += nwarps * W) {
    // row k * 32 + lane of the window: its extent and whether it is non-empty
    int64_t e0[kRowsPerLane], e1[kRowsPerLane];
    unsigned mask[kRowsPerLane];
    (void)mask;
#pragma unroll
    for (int k = 0; k < kRowsPerLane; ++k) {
      const int64_t i = base + k * 32 + lane;
      const bool ok = i < n;
      e0[k] = ok ? ld_stream(row_ptr + i, pf) : 0;
      e1[k] = ok ? ld_stream(row_ptr + i + 1, pf) : 0;
    }
    // compaction through shared memory: each non-empty row writes its (row,
    // extent) at its rank in the window; lane l then takes entries l, l + 32, ...
    int total = 0;
#pragma unroll
    for (int k = 0; k < kRowsPerLane; ++k) {
      mask[k] = __ballot_sync(0xffffffffu, e1[k] > e0[k]);
      if (e1[k] > e0[k]) {
        const int rank = total + __popc(mask[k] & lanemask_lt());
        crow[rank] = (int32_t)(k * 32 + lane);
        ce0[rank] = e0[k];
        ce1[rank] = e1[k];
      }
      total += __popc(mask[k]);
    }
    __syncwarp();
    for (int q = lane; q < total; q += 32)
      csr_row<SKETCH, GRAD, GSMEM, SC>(base + crow[q], ce0[q], ce1[q], d, col, val, row_offset, key, M, s, scale, SA,
                                       bvec, x, g, gs, pf, pl);
    __syncwarp();
  }
  if (GRAD && GSMEM) {
    __syncthreads();
    for (int c = threadIdx.x; c < d; c += blockDim.x) {
      const double t = gs[c];
      if (t != 0.0) atomicAdd(&g[c], t);
    }
  }
}

template <bool SKETCH, bool GRAD, int SC>
void launch_sc(int grid, int64_t n, int d, const int64_t *row_ptr, const int32_t *col, const double *val,
               int64_t row_offset, uint64_t key, uint32_t M, int s, double scale, double *SA, const double *bvec,
               const double *x, double *g, cudaStream_t st) {
  const size_t smem = (size_t)d * 8;
  if (GRAD && smem <= 96 * 1024) {
    IHS_SMEM_ATTR((csr_sketch_grad_kernel<SKETCH, GRAD, true, SC>), smem);
    csr_sketch_grad_kernel<SKETCH, GRAD, true, SC><<<grid, 256, smem, st>>>(n, d, row_ptr, col, val, row_offset, key,
                                                                           M, s, scale, SA, bvec, x, g);
  } else {
    csr_sketch_grad_kernel<SKETCH, GRAD, false, SC><<<grid, 256, 0, st>>>(n, d, row_ptr, col, val, row_offset, key,
                                                                         M, s, scale, SA, bvec, x, g);
  }
}

template <bool SKETCH, bool GRAD>
void launch_t(int grid, int64_t n, int d, const int64_t *row_ptr, const int32_t *col, const double *val,
              int64_t row_offset, uint64_t key, uint32_t M, int s, double scale, double *SA, const double *bvec,
              const double *x, double *g, cudaStream_t st) {
  switch (SKETCH ? s : 1) {
    case 1: launch_sc<SKETCH, GRAD, 1>(grid, n, d, row_ptr, col, val, row_offset, key, M, s, scale, SA, bvec, x, g, st); break;
    case 2: launch_sc<SKETCH, GRAD, 2>(grid, n, d, row_ptr, col, val, row_offset, key, M, s, scale, SA, bvec, x, g, st); break;
    case 4: launch_sc<SKETCH, GRAD, 4>(grid, n, d, row_ptr, col, val, row_offset, key, M, s, scale, SA, bvec, x, g, st); break;
    case 8: launch_sc<SKETCH, GRAD, 8>(grid, n, d, row_ptr, col, val, row_offset, key, M, s, scale, SA, bvec, x, g, st); break;
    default: launch_sc<SKETCH, GRAD, 0>(grid, n, d, row_ptr, col, val, row_offset, key, M, s, scale, SA, bvec, x, g, st);
  }
}
}  // namespace

cudaError_t launch_csr_sketch_grad(int64_t n, int64_t d, const int64_t *row_ptr, const int32_t *col,
                                   const double *val, int64_t row_offset, uint64_t key, int64_t m, int s,
                                   double scale, double *SA, const double *bvec, const double *x, double *g,
                                   cudaStream_t st, LaunchCounter lc) {
  if (n <= 0) return cudaSuccess;
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
  const uint32_t M = (uint32_t)(m / s);
  const bool sk = SA != nullptr, gr = g != nullptr;
  if (sk && gr) launch_t<true, true>(grid, n, (int)d, row_ptr, col, val, row_offset, key, M, s, scale, SA, bvec, x, g, st);
  else if (sk) launch_t<true, false>(grid, n, (int)d, row_ptr, col, val, row_offset, key, M, s, scale, SA, bvec, x, g, st);
  else if (gr) launch_t<false, true>(grid, n, (int)d, row_ptr, col, val, row_offset, key, M, s, scale, SA, bvec, x, g, st);
  lc.add();
  return cudaGetLastError();
}

}  // namespace ihs
