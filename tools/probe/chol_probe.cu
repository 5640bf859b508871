// Microbenchmark (not product code): clocks per call of the 32x32 Cholesky
// building blocks, rotated (chol_blocks.cuh) vs fully unrolled, plus the
// latency of the primitives on their critical path.  One CTA, clock64().
#include <cstdio>
#include <utility>
#include <cuda_runtime.h>
#include "../../paper_1910_14166_b200/csrc/chol_blocks.cuh"

using namespace ihs;
constexpr int LD = 36;

template <int J>
__device__ __forceinline__ void u_diag_step(double (&row)[32], int lane, bool &bad, double *rd) {
  const double piv = __shfl_sync(0xffffffffu, row[J], J);
  bad |= !(piv > 0.0);
  double sq, r;
  pivot_rsqrt(piv, sq, r);
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
__device__ __forceinline__ void u_diag(double (&row)[32], int lane, bool &bad, double *rd, std::integer_sequence<int, Js...>) {
  (u_diag_step<Js>(row, lane, bad, rd), ...);
}
template <int J>
__device__ __forceinline__ void u_trsm_step(double (&xr)[32], const double *rd, const double *L11, int lda) {
  const double xj = xr[J] * rd[J];
  xr[J] = xj;
#pragma unroll
  for (int k = J + 1; k < 32; ++k) xr[k] -= xj * L11[k * lda + J];
}
template <int... Js>
__device__ __forceinline__ void u_trsm(double (&xr)[32], const double *rd, const double *L11, int lda, std::integer_sequence<int, Js...>) {
  (u_trsm_step<Js>(xr, rd, L11, lda), ...);
}

// v4: unrolled; the next pivot's own update uses the lane's local l_ij (no
// shuffle on the pivot chain), and the pivot is broadcast from that register.
template <int J>
__device__ __forceinline__ void v4_step(double (&row)[32], int lane, bool &bad, double *rd, double &pnext) {
  const double piv = __shfl_sync(0xffffffffu, pnext, J);
  bad |= !(piv > 0.0);
  double sq, r;
  pivot_rsqrt(piv, sq, r);
  const double lij = (lane > J) ? row[J] * r : (lane == J ? sq : 0.0);
  row[J] = lij;
  if (lane == 0) rd[J] = r;
  if constexpr (J + 1 < 32) pnext = fma(-lij, lij, row[J + 1]);  // valid on lane J+1 only
#pragma unroll
  for (int k = J + 1; k < 32; ++k) {
    const double lkj = __shfl_sync(0xffffffffu, lij, k);
    if (lane >= k) row[k] -= lij * lkj;
  }
}
template <int... Js>
__device__ __forceinline__ void v4_diag(double (&row)[32], int lane, bool &bad, double *rd, std::integer_sequence<int, Js...>) {
  double pnext = row[0];
  (v4_step<Js>(row, lane, bad, rd, pnext), ...);
}

// v5: unconditional updates (entries right of the diagonal pick up unused values)
template <int J>
__device__ __forceinline__ void v5_step(double (&row)[32], int lane, bool &bad, double *rd) {
  const double piv = __shfl_sync(0xffffffffu, row[J], J);
  bad |= !(piv > 0.0);
  double sq, r;
  pivot_rsqrt(piv, sq, r);
  const double lij = (lane > J) ? row[J] * r : (lane == J ? sq : 0.0);
  row[J] = lij;
  if (lane == 0) rd[J] = r;
#pragma unroll
  for (int k = J + 1; k < 32; ++k) row[k] = fma(-lij, __shfl_sync(0xffffffffu, lij, k), row[k]);
}
template <int... Js>
__device__ __forceinline__ void v5_diag(double (&row)[32], int lane, bool &bad, double *rd, std::integer_sequence<int, Js...>) {
  (v5_step<Js>(row, lane, bad, rd), ...);
}
// v6: lkj broadcast through shared memory (one STS of the column, LDS broadcasts)
template <int J>
__device__ __forceinline__ void v6_step(double (&row)[32], int lane, bool &bad, double *rd, double *col) {
  const double piv = __shfl_sync(0xffffffffu, row[J], J);
  bad |= !(piv > 0.0);
  double sq, r;
  pivot_rsqrt(piv, sq, r);
  const double lij = (lane > J) ? row[J] * r : (lane == J ? sq : 0.0);
  row[J] = lij;
  if (lane == 0) rd[J] = r;
  col[(J & 1) * 32 + lane] = lij;
  __syncwarp();
#pragma unroll
  for (int k = J + 1; k < 32; ++k) row[k] = fma(-lij, col[(J & 1) * 32 + k], row[k]);
}
template <int... Js>
__device__ __forceinline__ void v6_diag(double (&row)[32], int lane, bool &bad, double *rd, double *col, std::integer_sequence<int, Js...>) {
  (v6_step<Js>(row, lane, bad, rd, col), ...);
}

__device__ void load_spd(double *B) {
  // B = I*40 + ones (SPD), lower part
  for (int e = threadIdx.x; e < 32 * LD; e += blockDim.x) {
    int i = e / LD, c = e % LD;
    B[e] = (c < 32) ? (1.0 + (i == c ? 40.0 : 0.0)) : 0.0;
  }
}

__global__ void k_chol(int variant, int reps, long long *out, double *sink) {
  __shared__ double B[32 * LD];
  __shared__ double rd[32];
  __shared__ double X[128 * 33];
  const int lane = threadIdx.x & 31;
  long long t_total = 0;
  for (int rep = 0; rep < reps; ++rep) {
    load_spd(B);
    for (int e = threadIdx.x; e < 128 * 33; e += blockDim.x) X[e] = 1.0 + (e % 7);
    __syncthreads();
    long long t0 = clock64();
    if (variant == 0 && threadIdx.x < 32) {
      __shared__ double cb[64];
      warp_chol32(B, LD, rd, 32, cb);
    } else if (variant == 1 && threadIdx.x < 32) {
      double row[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) row[c] = (c <= lane) ? B[lane * LD + c] : 0.0;
      bool bad = false;
      u_diag(row, lane, bad, rd, std::make_integer_sequence<int, 32>{});
#pragma unroll
      for (int c = 0; c < 32; ++c)
        if (c <= lane) B[lane * LD + c] = row[c];
    } else if (variant == 4 && threadIdx.x < 32) {
      double row[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) row[c] = (c <= lane) ? B[lane * LD + c] : 0.0;
      bool bad = false;
      v4_diag(row, lane, bad, rd, std::make_integer_sequence<int, 32>{});
#pragma unroll
      for (int c = 0; c < 32; ++c)
        if (c <= lane) B[lane * LD + c] = row[c];
    } else if ((variant == 5 || variant == 6) && threadIdx.x < 32) {
      __shared__ double colbuf[64];
      double row[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) row[c] = (c <= lane) ? B[lane * LD + c] : 0.0;
      bool bad = false;
      if (variant == 5) v5_diag(row, lane, bad, rd, std::make_integer_sequence<int, 32>{});
      else v6_diag(row, lane, bad, rd, colbuf, std::make_integer_sequence<int, 32>{});
#pragma unroll
      for (int c = 0; c < 32; ++c)
        if (c <= lane) B[lane * LD + c] = row[c];
    } else if (variant == 2) {
      thread_trsm32(X + threadIdx.x * 33, B, LD, rd);
    } else if (variant == 3) {
      double xr[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) xr[c] = X[threadIdx.x * 33 + c];
      u_trsm(xr, rd, B, LD, std::make_integer_sequence<int, 32>{});
#pragma unroll
      for (int c = 0; c < 32; ++c) X[threadIdx.x * 33 + c] = xr[c];
    }
    __syncthreads();
    t_total += clock64() - t0;
  }
  if (threadIdx.x == 0) out[variant] = t_total / reps;
  if (threadIdx.x == 0) sink[0] = B[5] + X[7];
}

// primitive latencies (single thread chain)
__global__ void k_prim(long long *out, double seed) {
  double x = seed;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) x = fma(x, 1.0000001, 1e-9);
  long long t1 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) x = rsqrt(x) + 1.0;
  long long t2 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) x = __shfl_sync(0xffffffffu, x, (i + threadIdx.x) & 31) + 1.0;
  long long t3 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) x = sqrt(x) + 1.0;
  long long t4 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) x = 1.0 / x + 1.0;
  long long t5 = clock64();
  if (threadIdx.x == 0) {
    out[0] = (t1 - t0) / 256;
    out[1] = (t2 - t1) / 256;
    out[2] = (t3 - t2) / 256;
    out[3] = (t4 - t3) / 256;
    out[4] = (t5 - t4) / 256;
  }
  if (x == 12345.0) out[5] = 1;
}

int main() {
  long long *d_out, h[8];
  double *sink;
  cudaMalloc(&d_out, 64);
  cudaMalloc(&sink, 64);
  const char *names[] = {"warp_chol32 (rotated)", "diag unrolled", "thread_trsm32 x128 thr (rotated)",
                         "trsm unrolled x128 thr", "diag unrolled, local next pivot", "diag unconditional fma",
                         "diag smem column broadcast"};
  for (int v = 0; v < 7; ++v) {
    int threads = (v < 2 || v >= 4) ? 32 : 128;
    k_chol<<<1, threads>>>(v, 20, d_out, sink);  // warm (i-cache)
    k_chol<<<1, threads>>>(v, 20, d_out, sink);
    cudaMemcpy(h, d_out, 64, cudaMemcpyDeviceToHost);
    printf("%-34s %lld clk/call\n", names[v], h[v]);
  }
  k_prim<<<1, 32>>>(d_out, 1.5);
  cudaMemcpy(h, d_out, 64, cudaMemcpyDeviceToHost);
  printf("latency: dfma %lld, rsqrt+add %lld, shfl+add %lld, sqrt+add %lld, div+add %lld clk\n", h[0], h[1], h[2], h[3],
         h[4]);
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
