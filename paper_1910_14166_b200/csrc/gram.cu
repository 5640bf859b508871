// a4: H = (SA)^T SA, the approximate Hessian (section 1;
// O(m d^2)), the one dense contraction of the path.  fp64 on
// the DMMA tensor pipe (mma.sync m8n8k4 f64 -> DMMA.8x8x4; tcgen05 has no f64
// kind on sm_100a).  Only upper-triangular 64x64 tiles are computed (symmetry
// halves the flops); split-K partials are summed in a fixed order and mirrored.
#include "common.cuh"
#include "kernels.h"

namespace ihs {

namespace {
constexpr int GT = 64;       // CTA tile edge
constexpr int KC = 32;       // rows of SA per smem stage
constexpr int LDS = GT + 4;  // padded row stride (== 4 mod 16 doubles: conflict-free fragments)
constexpr int kStagesK = 2;  // stream-K kernel: double-buffered stages (3 measured slower on C3: 0.333 vs 0.324 ms)

__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void tri_decode(int t, int tiles, int &P, int &Q) {
  // row-major enumeration of {(P, Q): P <= Q}
  int p = 0, rem = t;
  while (rem >= tiles - p) {
    rem -= tiles - p;
    ++p;
  }
  P = p;
  Q = p + rem;
}

__device__ __forceinline__ void cp_async8(double *smem, const double *gmem, bool pred) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  int sz = pred ? 8 : 0;  // zero-fill when out of range
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(sa), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

// 4 warps; warp (wm, wn) owns the 32x32 sub-tile [32wm, +32) x [32wn, +32) as
// 4x4 DMMA 8x8 tiles.  Double-buffered cp.async stages of KC rows.
__global__ void __launch_bounds__(128) gram_kernel(const double *__restrict__ SA, int64_t m, int d, int tiles,
                                                   int ntri, int64_t kchunk, double *__restrict__ partials) {
  extern __shared__ double sm[];
  double *Xp = sm;                   // [2][KC][LDS]
  double *Xq = sm + 2 * KC * LDS;    // [2][KC][LDS]
  int P, Q;
  tri_decode(blockIdx.x, tiles, P, Q);
  const bool diag = (P == Q);
  const int64_t k0 = (int64_t)blockIdx.y * kchunk;
  const int64_t k1 = min(m, k0 + kchunk);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  auto load_stage = [&](int buf, int64_t kb) {
    // KC x 64 doubles per matrix: 2048 / 128 threads = 16 each
#pragma unroll
    for (int it = 0; it < (KC * GT) / 128; ++it) {
      int e = it * 128 + tid;
      int r = e / GT, c = e % GT;
      int64_t row = kb + r;
      bool rin = row < k1;
      int cp = P * GT + c, cq = Q * GT + c;
      cp_async8(&Xp[(buf * KC + r) * LDS + c], SA + (rin ? row : 0) * d + (cp < d ? cp : 0), rin && cp < d);
      if (!diag) cp_async8(&Xq[(buf * KC + r) * LDS + c], SA + (rin ? row : 0) * d + (cq < d ? cq : 0), rin && cq < d);
    }
    cp_async_commit();
  };

  const int nstages = (int)((k1 - k0 + KC - 1) / KC);
  if (nstages > 0) load_stage(0, k0);
  for (int s = 0; s < nstages; ++s) {
    const int buf = s & 1;
    if (s + 1 < nstages) {
      load_stage(buf ^ 1, k0 + (int64_t)(s + 1) * KC);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double *xp = Xp + buf * KC * LDS;
    const double *xq = (diag ? Xp : Xq) + buf * KC * LDS;
#pragma unroll
    for (int kk = 0; kk < KC; kk += 4) {
      const int kr = kk + (lane & 3);
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = xp[kr * LDS + 32 * wm + 8 * i + (lane >> 2)];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = xq[kr * LDS + 32 * wn + 8 * j + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
    __syncthreads();
  }
  double *out = partials + ((int64_t)blockIdx.y * ntri + blockIdx.x) * (GT * GT);
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int r = 32 * wm + 8 * i + (lane >> 2);
      int c = 32 * wn + 8 * j + 2 * (lane & 3);
      out[r * GT + c] = acc[i][j][0];
      out[r * GT + c + 1] = acc[i][j][1];
    }
}

// H[p][q] = H[q][p] = scale^2 * sum_split partial (fixed order).  One thread
// per element of the upper tiles (grid: tile x 16 chunks of 256 elements).
__global__ void __launch_bounds__(256) gram_reduce_kernel(const double *__restrict__ partials, int d, int tiles,
                                                          int ntri, int nsplit, double scale2,
                                                          double *__restrict__ H) {
  int P, Q;
  tri_decode(blockIdx.x, tiles, P, Q);
  const int e = blockIdx.y * 256 + threadIdx.x;
  const int r = e / GT, c = e % GT;
  const int p = P * GT + r, q = Q * GT + c;
  if (p >= d || q >= d) return;
  if (P == Q && q < p) return;
  const double *src = partials + (int64_t)blockIdx.x * (GT * GT) + e;
  const int64_t stride = (int64_t)ntri * (GT * GT);
  double s = 0.0;
#pragma unroll 8
  for (int k = 0; k < nsplit; ++k) s += src[k * stride];
  s *= scale2;
  H[(int64_t)p * d + q] = s;
  H[(int64_t)q * d + p] = s;
}
// ---------------------------------------------------------------------------
// Stream-K variant for many tiles (d >= 384; C3: 136 upper tiles, m = 8192):
// the (tile, k-chunk) items, tile-major, are dealt out in equal contiguous
// ranges to a persistent grid of 2 CTAs per SM, so every SM does the same
// number of DMMAs (the split-K grid left ~8% of the SMs half idle).  A CTA
// keeps its accumulators while consecutive items belong to the same tile and
// flushes a partial tile (at most two per CTA: a range is shorter than a
// tile's chunk count) with its tile id; the reduction sums, per tile, the
// partials of the CTAs that covered it in CTA order (fixed, deterministic).
// Stages are loaded with 16-byte cp.async (d even, 16-byte aligned SA).
__device__ __forceinline__ void cp_async16(double *smem, const double *gmem, bool pred) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  int sz = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(gmem), "r"(sz));
}
// The same with an L2 eviction policy (the look-ahead Gram beside a CSR pass
// reads SA evict_first, so the pass's L2-resident reductions stay in L2).
__device__ __forceinline__ void cp_async16_hint(double *smem, const double *gmem, bool pred, uint64_t pol) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  int sz = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2, %3;" ::"r"(sa), "l"(gmem), "r"(sz),
               "l"(pol));
}

__global__ void __launch_bounds__(128) gram_streamk_kernel(const double *__restrict__ SA, int64_t m, int d,
                                                           int tiles, int ntri, int kch, int ipc,
                                                           double *__restrict__ partials, int *__restrict__ slot_tile,
                                                           int hint) {
  extern __shared__ double sm[];
  double *Xp = sm;                         // [kStagesK][KC][LDS]
  double *Xq = sm + kStagesK * KC * LDS;  // [kStagesK][KC][LDS]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1;
  const int64_t total = (int64_t)ntri * kch;
  const int64_t i0 = (int64_t)blockIdx.x * ipc, i1 = min(total, i0 + ipc);
  if (tid == 0) slot_tile[2 * blockIdx.x] = slot_tile[2 * blockIdx.x + 1] = -1;
  uint64_t pol = 0;
  if (hint) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  double acc[4][4][2];
  int cur = -1, slot = 0;
  auto flush = [&]() {
    double *out = partials + ((int64_t)blockIdx.x * 2 + slot) * (GT * GT);
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int r = 32 * wm + 8 * i + (lane >> 2);
        const int c = 32 * wn + 8 * j + 2 * (lane & 3);
        out[r * GT + c] = acc[i][j][0];
        out[r * GT + c + 1] = acc[i][j][1];
      }
    if (tid == 0) slot_tile[2 * blockIdx.x + slot] = cur;
    ++slot;
  };
  for (int64_t it = i0; it < i1; ++it) {
    const int tile = (int)(it / kch), kc = (int)(it % kch);
    if (tile != cur) {
      if (cur >= 0) flush();
      cur = tile;
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    }
    int P, Q;
    tri_decode(tile, tiles, P, Q);
    const bool diag = (P == Q);
    const int64_t k0 = m * kc / kch, k1 = m * (kc + 1) / kch;
    auto load_stage = [&](int buf, int64_t kb) {
      // KC x 64 doubles per matrix in 16-byte pieces: 1024 / 128 threads = 8 each
#pragma unroll
      for (int t2 = 0; t2 < (KC * GT / 2) / 128; ++t2) {
        const int e = t2 * 128 + tid;
        const int r = e / (GT / 2), c = 2 * (e % (GT / 2));
        const int64_t row = kb + r;
        const bool rin = row < k1;
        const int cp = P * GT + c, cq = Q * GT + c;
        const double *gp = SA + (rin ? row : 0) * d + (cp < d ? cp : 0);
        const double *gq = SA + (rin ? row : 0) * d + (cq < d ? cq : 0);
        if (hint) {
          cp_async16_hint(&Xp[(buf * KC + r) * LDS + c], gp, rin && cp < d, pol);
          if (!diag) cp_async16_hint(&Xq[(buf * KC + r) * LDS + c], gq, rin && cq < d, pol);
        } else {
          cp_async16(&Xp[(buf * KC + r) * LDS + c], gp, rin && cp < d);
          if (!diag) cp_async16(&Xq[(buf * KC + r) * LDS + c], gq, rin && cq < d);
        }
      }
      cp_async_commit();
    };
    const int nstages = (int)((k1 - k0 + KC - 1) / KC);
    if (nstages > 0) load_stage(0, k0);
    for (int s2 = 0; s2 < nstages; ++s2) {
      const int buf = s2 & 1;
      if (s2 + 1 < nstages) {
        load_stage(buf ^ 1, k0 + (int64_t)(s2 + 1) * KC);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
      const double *xp = Xp + buf * KC * LDS;
      const double *xq = (diag ? Xp : Xq) + buf * KC * LDS;
#pragma unroll
      for (int kk = 0; kk < KC; kk += 4) {
        const int kr = kk + (lane & 3);
        double a[4], b[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = xp[kr * LDS + 32 * wm + 8 * i + (lane >> 2)];
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = xq[kr * LDS + 32 * wn + 8 * j + (lane >> 2)];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
      }
      __syncthreads();
    }
  }
  if (cur >= 0) flush();
}

// Per tile: sum the partials of the CTAs whose item range covered it (CTA
// order), scale^2, mirror.  grid: tile x 16 chunks of 256 elements.
__global__ void __launch_bounds__(256) gram_streamk_reduce_kernel(const double *__restrict__ partials,
                                                                  const int *__restrict__ slot_tile, int d, int tiles,
                                                                  int kch, int ipc, double scale2,
                                                                  double *__restrict__ H) {
  const int t = blockIdx.x;
  int P, Q;
  tri_decode(t, tiles, P, Q);
  const int e = blockIdx.y * 256 + threadIdx.x;
  const int r = e / GT, c = e % GT;
  const int p = P * GT + r, q = Q * GT + c;
  if (p >= d || q >= d) return;
  if (P == Q && q < p) return;
  const int64_t c0 = ((int64_t)t * kch) / ipc, c1 = ((int64_t)t * kch + kch - 1) / ipc;
  double s = 0.0;
  for (int64_t cta = c0; cta <= c1; ++cta) {
    const int sl = slot_tile[2 * cta] == t ? 0 : 1;
    s += partials[((int64_t)cta * 2 + sl) * (GT * GT) + e];
  }
  s *= scale2;
  H[(int64_t)p * d + q] = s;
  H[(int64_t)q * d + p] = s;
}

// ---------------------------------------------------------------------------
// Stream-K with 128 x 128 tiles for large d (d >= 512: C3's 36 upper tiles):
// half the L2 operand reads of the 64 x 64 tiles (each CTA tile reads 2 x 128
// columns of SA per k-row for 128 x 128 outputs) -- the look-ahead Gram runs
// beside the CSR pass, which is bound by its L2 reductions -- and the same
// DMMAs per shared-memory fragment load as the 64 tiles.  16 warps,
// warp (wm, wn) owns rows [32 wm, +32) x columns [32 wn, +32) as 4 x 4 DMMA
// 8 x 8 tiles (32 fp64 accumulators a thread: no spills, unlike a 32 x 64
// warp tile at 8 warps); one CTA per SM; kStages2 stages of KC2 rows.
constexpr int GT2 = 128;
constexpr int KC2 = 16;
constexpr int LDS2 = GT2 + 4;  // == 4 mod 16 doubles: conflict-free fragment loads
constexpr int kStages2 = 3;

__global__ void __launch_bounds__(512, 1) gram_streamk128_kernel(const double *__restrict__ SA, int64_t m, int d,
                                                                 int tiles, int ntri, int kch, int ipc,
                                                                 double *__restrict__ partials,
                                                                 int *__restrict__ slot_tile, int hint) {
  extern __shared__ double sm[];
  double *Xp = sm;                          // [kStages2][KC2][LDS2]
  double *Xq = sm + kStages2 * KC2 * LDS2;  // [kStages2][KC2][LDS2]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 2, wn = warp & 3;  // 16 warps: 4 x 4 of 32 x 32
  const int64_t total = (int64_t)ntri * kch;
  const int64_t i0 = (int64_t)blockIdx.x * ipc, i1 = min(total, i0 + ipc);
  if (tid == 0) slot_tile[2 * blockIdx.x] = slot_tile[2 * blockIdx.x + 1] = -1;
  uint64_t pol = 0;
  if (hint) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  double acc[4][4][2];
  int cur = -1, slot = 0;
  auto flush = [&]() {
    double *out = partials + ((int64_t)blockIdx.x * 2 + slot) * (GT2 * GT2);
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int r = 32 * wm + 8 * i + (lane >> 2);
        const int c = 32 * wn + 8 * j + 2 * (lane & 3);
        *reinterpret_cast<double2 *>(out + r * GT2 + c) = make_double2(acc[i][j][0], acc[i][j][1]);
      }
    if (tid == 0) slot_tile[2 * blockIdx.x + slot] = cur;
    ++slot;
  };
  for (int64_t it = i0; it < i1; ++it) {
    const int tile = (int)(it / kch), kc = (int)(it % kch);
    if (tile != cur) {
      if (cur >= 0) flush();
      cur = tile;
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    }
    int P, Q;
    tri_decode(tile, tiles, P, Q);
    const bool diag = (P == Q);
    const int64_t k0 = m * kc / kch, k1 = m * (kc + 1) / kch;
    auto load_stage = [&](int buf, int64_t kb) {
      // KC2 x 128 doubles per matrix in 16-byte pieces: 1024 / 512 threads = 2 each
#pragma unroll
      for (int t2 = 0; t2 < (KC2 * GT2 / 2) / 512; ++t2) {
        const int e = t2 * 512 + tid;
        const int r = e / (GT2 / 2), c = 2 * (e % (GT2 / 2));
        const int64_t row = kb + r;
        const bool rin = row < k1;
        const int cp = P * GT2 + c, cq = Q * GT2 + c;
        const double *gp = SA + (rin ? row : 0) * d + (cp < d ? cp : 0);
        const double *gq = SA + (rin ? row : 0) * d + (cq < d ? cq : 0);
        if (hint) {
          cp_async16_hint(&Xp[(buf * KC2 + r) * LDS2 + c], gp, rin && cp < d, pol);
          if (!diag) cp_async16_hint(&Xq[(buf * KC2 + r) * LDS2 + c], gq, rin && cq < d, pol);
        } else {
          cp_async16(&Xp[(buf * KC2 + r) * LDS2 + c], gp, rin && cp < d);
          if (!diag) cp_async16(&Xq[(buf * KC2 + r) * LDS2 + c], gq, rin && cq < d);
        }
      }
      cp_async_commit();
    };
    const int nstages = (int)((k1 - k0 + KC2 - 1) / KC2);
    // prologue: kStages2 - 1 stages in flight (empty groups keep the count uniform)
#pragma unroll
    for (int q = 0; q < kStages2 - 1; ++q) {
      if (q < nstages)
        load_stage(q, k0 + (int64_t)q * KC2);
      else
        cp_async_commit();
    }
    for (int s2 = 0; s2 < nstages; ++s2) {
      cp_async_wait<kStages2 - 2>();
      __syncthreads();
      const int nxt = s2 + kStages2 - 1;
      if (nxt < nstages)
        load_stage(nxt % kStages2, k0 + (int64_t)nxt * KC2);
      else
        cp_async_commit();
      const int buf = s2 % kStages2;
      const double *xp = Xp + buf * KC2 * LDS2;
      const double *xq = (diag ? Xp : Xq) + buf * KC2 * LDS2;
      // a diagonal tile's warps wholly below the diagonal skip their DMMAs
      // (the reduction reads the upper triangle only)
      if (!(diag && wm > wn))
#pragma unroll
      for (int kk = 0; kk < KC2; kk += 4) {
        const int kr = kk + (lane & 3);
        double a[4], b[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = xp[kr * LDS2 + 32 * wm + 8 * i + (lane >> 2)];
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = xq[kr * LDS2 + 32 * wn + 8 * j + (lane >> 2)];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
      }
    }
    cp_async_wait<0>();
    __syncthreads();
  }
  if (cur >= 0) flush();
}

// Per 128-tile: the partials of the CTAs that covered it, in CTA order; scale^2, mirror.
// grid: tile x 64 chunks of 256 elements.
__global__ void __launch_bounds__(256) gram_streamk128_reduce_kernel(const double *__restrict__ partials,
                                                                     const int *__restrict__ slot_tile, int d,
                                                                     int tiles, int kch, int ipc, double scale2,
                                                                     double *__restrict__ H) {
  const int t = blockIdx.x;
  int P, Q;
  tri_decode(t, tiles, P, Q);
  const int e = blockIdx.y * 256 + threadIdx.x;
  const int r = e / GT2, c = e % GT2;
  const int p = P * GT2 + r, q = Q * GT2 + c;
  if (p >= d || q >= d) return;
  if (P == Q && q < p) return;
  const int64_t c0 = ((int64_t)t * kch) / ipc, c1 = ((int64_t)t * kch + kch - 1) / ipc;
  double s = 0.0;
  for (int64_t cta = c0; cta <= c1; ++cta) {
    const int sl = slot_tile[2 * cta] == t ? 0 : 1;
    s += partials[((int64_t)cta * 2 + sl) * (GT2 * GT2) + e];
  }
  s *= scale2;
  H[(int64_t)p * d + q] = s;
  H[(int64_t)q * d + p] = s;
}

}  // namespace

GramPlan gram_plan(int64_t m, int64_t d, int num_sms, int ctas_per_sm, bool beside) {
  GramPlan p;
  p.m = m;
  p.d = d;
  p.tiles = (int)((d + GT - 1) / GT);
  p.ntri = p.tiles * (p.tiles + 1) / 2;
  // split K so that ~2 waves of CTAs run, with at least 2 stages per CTA
  int64_t want = std::max<int64_t>(1, (2 * (int64_t)num_sms + p.ntri - 1) / p.ntri);
  int64_t maxsplit = std::max<int64_t>(1, (m + 2 * KC - 1) / (2 * KC));
  int64_t ns = std::min(want, maxsplit);
  int64_t kc = (m + ns - 1) / ns;
  kc = (kc + KC - 1) / KC * KC;
  p.kchunk = std::max<int64_t>(kc, KC);
  p.nsplit = (int)std::max<int64_t>(1, (m + p.kchunk - 1) / p.kchunk);
  // stream-K for many tiles: 2 CTAs per SM, k-chunks per tile chosen so that
  // the items divide as evenly as possible over the CTAs (>= 64 rows a chunk)
  if (p.ntri >= 16 && d % 2 == 0 && m >= 256) {
    const int64_t ncta = (int64_t)ctas_per_sm * num_sms;
    const int64_t kmin = std::max<int64_t>(1, (2 * ncta + p.ntri - 1) / p.ntri);
    const int64_t kmax = std::max<int64_t>(kmin, m / 64);
    int64_t best = kmin;
    double best_waste = 1e30;
    for (int64_t k = kmin; k <= kmax && k <= 8 * kmin; ++k) {
      const int64_t tot = p.ntri * k, ipc = (tot + ncta - 1) / ncta;
      const double waste = (double)(ipc * ncta - tot) / (double)tot;
      if (waste < best_waste - 1e-9) {
        best_waste = waste;
        best = k;
      }
    }
    p.kch = (int)best;
    p.ipc = (int)((p.ntri * best + ncta - 1) / ncta);
    p.ncta = (int)((p.ntri * best + p.ipc - 1) / p.ipc);
    if (p.ipc > p.kch) p.ncta = 0;  // a CTA would span three tiles: keep split-K
  }
  // 128 x 128 tiles (one CTA per SM) for d >= 512 when the Gram runs BESIDE
  // another kernel (the look-ahead Gram next to the CSR pass, C3): alone it
  // is slower than the 64 x 64 stream-K (0.357 vs 0.322 ms: one CTA of 8
  // warps per SM hides less latency), beside the pass it leaves the pass's
  // CTAs room and halves the L2 operand reads (C3 step 0.631 -> 0.426 ms)
  if (beside && p.ncta > 0 && d >= 512 && num_sms >= 64 && m >= 1024) {
    const int t2 = (int)((d + GT2 - 1) / GT2);
    const int64_t ntri2 = (int64_t)t2 * (t2 + 1) / 2;
    const int64_t ncta = num_sms;
    const int64_t kmin = std::max<int64_t>(1, (2 * ncta + ntri2 - 1) / ntri2);
    const int64_t kmax = std::max<int64_t>(kmin, m / 64);
    int64_t best = kmin;
    double best_waste = 1e30;
    for (int64_t k = kmin; k <= kmax && k <= 8 * kmin; ++k) {
      const int64_t tot = ntri2 * k, ipc = (tot + ncta - 1) / ncta;
      const double waste = (double)(ipc * ncta - tot) / (double)tot;
      if (waste < best_waste - 1e-9) {
        best_waste = waste;
        best = k;
      }
    }
    const int ipc2 = (int)((ntri2 * best + ncta - 1) / ncta);
    if (ipc2 <= best) {
      p.gt = GT2;
      p.tiles = t2;
      p.ntri = (int)ntri2;
      p.kch = (int)best;
      p.ipc = ipc2;
      p.ncta = (int)((ntri2 * best + ipc2 - 1) / ipc2);
    }
  }
  return p;
}

cudaError_t launch_gram(const GramPlan &p, const double *SA, double scale, double *partials, double *H,
                        cudaStream_t st, LaunchCounter lc, int hint) {
  const size_t smem = (size_t)4 * KC * LDS * 8;
  if (p.gt == GT2 && p.ncta > 0 && (reinterpret_cast<uintptr_t>(SA) % 16) == 0) {
    const size_t smem2 = (size_t)2 * kStages2 * KC2 * LDS2 * 8;
    IHS_SMEM_ATTR(gram_streamk128_kernel, smem2);
    int *slot_tile = reinterpret_cast<int *>(partials + (size_t)p.ncta * 2 * GT2 * GT2);
    gram_streamk128_kernel<<<p.ncta, 512, smem2, st>>>(SA, p.m, (int)p.d, p.tiles, p.ntri, p.kch, p.ipc, partials,
                                                       slot_tile, hint);
    gram_streamk128_reduce_kernel<<<dim3(p.ntri, (GT2 * GT2) / 256), 256, 0, st>>>(
        partials, slot_tile, (int)p.d, p.tiles, p.kch, p.ipc, scale * scale, H);
    lc.add(2);
    return cudaGetLastError();
  }
  if (p.ncta > 0 && (reinterpret_cast<uintptr_t>(SA) % 16) == 0) {
    const size_t smem_sk = (size_t)2 * kStagesK * KC * LDS * 8;
    IHS_SMEM_ATTR(gram_streamk_kernel, smem_sk);
    int *slot_tile = reinterpret_cast<int *>(partials + (size_t)p.ncta * 2 * GT * GT);
    gram_streamk_kernel<<<p.ncta, 128, smem_sk, st>>>(SA, p.m, (int)p.d, p.tiles, p.ntri, p.kch, p.ipc, partials,
                                                      slot_tile, hint);
    gram_streamk_reduce_kernel<<<dim3(p.ntri, (GT * GT) / 256), 256, 0, st>>>(partials, slot_tile, (int)p.d, p.tiles,
                                                                               p.kch, p.ipc, scale * scale, H);
    lc.add(2);
    return cudaGetLastError();
  }
  IHS_SMEM_ATTR(gram_kernel, smem);
  dim3 grid(p.ntri, p.nsplit);
  gram_kernel<<<grid, 128, smem, st>>>(SA, p.m, (int)p.d, p.tiles, p.ntri, p.kchunk, partials);
  gram_reduce_kernel<<<dim3(p.ntri, (GT * GT) / 256), 256, 0, st>>>(partials, (int)p.d, p.tiles, p.ntri, p.nsplit,
                                                                     scale * scale, H);
  lc.add(2);
  return cudaGetLastError();
}

}  // namespace ihs
