// a1 + the first half of a2 for dense CountSketch (s = 1): hash every local row
// and stable counting-sort the row ids by bucket, so the sketch kernel can sum
// each bucket's rows in ascending row order in registers (no atomics, the
// oracle's order).  Also the bit-exact hash export (ihs_hash).
//
// PAPER.md:175-177 (section 2, CountSketch: one +-1 per column at row h(i)) and
// PAPER.md:236-240 (streaming application: bucket h(i) accumulates +-row i).
#include "common.cuh"
#include "kernels.h"

#include <algorithm>
#include <cstdlib>

namespace ihs {

namespace {
constexpr int kHistThreads = 256;
constexpr int kScatterWarps = 8;
constexpr int kScanTile = 4096;  // entries per scan tile (1024 threads x 4)

__global__ void hash_export_kernel(uint64_t key, uint32_t s, uint32_t M, int64_t row_begin, int64_t count,
                                   int32_t *__restrict__ bucket, int8_t *__restrict__ sign) {
  int64_t total = count * (int64_t)s;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = e / s;
    uint32_t j = (uint32_t)(e - r * s);
    bool neg;
    uint32_t b = hash_bucket(key, (uint64_t)(row_begin + r), j, s, M, neg);
    bucket[e] = (int32_t)b;
    sign[e] = neg ? int8_t(-1) : int8_t(1);
  }
}

// Per-chunk bucket histogram, written bucket-major: hist[b * nchunks + chunk].
// CTA k handles chunks k, k + gridDim.x, ... (gridDim.x = nchunks by default;
// fewer, persistent CTAs with IHS_SORT_CTAS).
__global__ void __launch_bounds__(kHistThreads) cs_hist_kernel(int64_t n, int64_t chunk, int64_t nchunks,
                                                               uint32_t m, uint64_t key, int64_t row_offset,
                                                               uint32_t jb, uint32_t sb, int32_t *__restrict__ hist) {
  extern __shared__ int32_t cnt[];
  for (int64_t cb = blockIdx.x; cb < nchunks; cb += gridDim.x) {
    for (uint32_t b = threadIdx.x; b < m; b += blockDim.x) cnt[b] = 0;
    __syncthreads();
    const int64_t r0 = cb * chunk;
    const int64_t r1 = min(n, r0 + chunk);
    for (int64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
      bool neg;
      uint32_t b = hash_bucket(key, (uint64_t)(row_offset + r), jb, sb, m, neg) - jb * m;
      atomicAdd(&cnt[b], 1);
    }
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < m; b += blockDim.x) hist[(int64_t)b * nchunks + cb] = cnt[b];
    __syncthreads();
  }
}

// Exclusive scan, phase 1: each 4096-entry tile scanned locally in place; the
// tile total goes to tile_sums[tile].
__global__ void __launch_bounds__(1024) scan_tiles_kernel(int32_t *__restrict__ a, int64_t E,
                                                          int32_t *__restrict__ tile_sums) {
  __shared__ int32_t wsum[32];
  const int64_t base = blockIdx.x * (int64_t)kScanTile + threadIdx.x * 4;
  int32_t v[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) v[i] = (base + i < E) ? a[base + i] : 0;
  int32_t t = v[0] + v[1] + v[2] + v[3];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int32_t incl = t;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int32_t w = wsum[lane];
    int32_t wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int32_t y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    wsum[lane] = wi - w;  // exclusive warp offsets
    if (lane == 31) tile_sums[blockIdx.x] = wi;
  }
  __syncthreads();
  int32_t run = wsum[warp] + incl - t;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (base + i < E) a[base + i] = run;
    run += v[i];
  }
}

// Exclusive scan, phase 2: one CTA scans the tile sums; tile_sums[ntiles] = total.
__global__ void __launch_bounds__(1024) scan_sums_kernel(int32_t *__restrict__ s, int64_t ntiles) {
  __shared__ int32_t wsum[32];
  __shared__ int32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t base = 0; base < ntiles; base += 1024) {
    int64_t i = base + threadIdx.x;
    int32_t v = i < ntiles ? s[i] : 0;
    int32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      int32_t w = wsum[lane], wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int32_t y = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += y;
      }
      wsum[lane] = wi - w;
    }
    __syncthreads();
    int32_t c = carry;
    if (i < ntiles) s[i] = c + wsum[warp] + incl - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry = c + wsum[warp] + incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) s[ntiles] = carry;
}

__device__ __forceinline__ int32_t scanned_at(const int32_t *hist, const int32_t *tile_sums, int64_t e) {
  return hist[e] + tile_sums[e / kScanTile];
}

// Stable scatter of row ids: rows of a chunk are split over 8 warps in order;
// each warp caches the buckets of its rows in registers (kMaxGroups groups of
// 32), counts them with warp-private shared-memory atomics, and after a
// cross-warp exclusive scan per bucket places every row with one
// atomicAdd-return per (group, bucket) leader: a warp's shared-memory atomics
// complete in issue order, so positions follow ascending row order within
// every bucket (stable).
constexpr int kMaxGroups = 16;  // rows per warp sub-chunk <= 512
__device__ __forceinline__ void cs_scatter_chunk(
    int64_t cb, int64_t n, int64_t chunk, int64_t nchunks, uint32_t m, uint64_t key, int64_t row_offset, uint32_t jb,
    uint32_t sb, const int32_t *__restrict__ hist, const int32_t *__restrict__ tile_sums, uint32_t *__restrict__ perm,
    int keep) {
  extern __shared__ unsigned char smem_raw[];
  int32_t *base = reinterpret_cast<int32_t *>(smem_raw);            // m
  int32_t *wcnt = base + m;                                           // 8 * m
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint32_t e = threadIdx.x; e < kScatterWarps * m; e += blockDim.x) wcnt[e] = 0;
  __syncthreads();
  const int64_t r0 = cb * chunk;
  const int64_t r1 = min(n, r0 + chunk);
  const int64_t sub = chunk / kScatterWarps;
  const int64_t ws = r0 + warp * sub;
  const int64_t we = min(r1, ws + sub);
  int32_t *my = wcnt + (size_t)warp * m;
  const int nbits = 32 - __clz((int)max(m - 1, 1u));  // bucket < 2^nbits
  uint32_t bk[kMaxGroups];
  unsigned pm[kMaxGroups];  // peer masks of phase 1, reused by phase 2
#pragma unroll
  for (int q = 0; q < kMaxGroups; ++q) {
    const int64_t r = ws + 32 * q + lane;
    bool neg = false;
    uint32_t b = 0xffffffffu;
    if (ws + 32 * q < we && r < we) b = hash_bucket(key, (uint64_t)(row_offset + r), jb, sb, m, neg) - jb * m;
    else b = 0;
    bk[q] = b | (neg ? 0x80000000u : 0u);  // m < 2^31: bit 31 free for the sign
    if (ws + 32 * q < we) {
      const bool valid = r < we;
      const uint32_t bb = bk[q] & 0x7fffffffu;
      const unsigned mask = peers_by_ballot(bb, nbits, valid);
      pm[q] = mask;
      if (valid && lane == __ffs(mask) - 1) atomicAdd(&my[bb], __popc(mask));
    } else {
      pm[q] = 0u;
    }
  }
  __syncthreads();
  for (uint32_t b = threadIdx.x; b < m; b += blockDim.x) {
    base[b] = scanned_at(hist, tile_sums, (int64_t)b * nchunks + cb);
    int32_t acc = 0;
#pragma unroll
    for (int w = 0; w < kScatterWarps; ++w) {
      const int32_t t = wcnt[(size_t)w * m + b];
      wcnt[(size_t)w * m + b] = acc;
      acc += t;
    }
  }
  __syncthreads();
  const unsigned lt = lanemask_lt();
  uint64_t pol = 0;
  if (keep) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
#pragma unroll
  for (int q = 0; q < kMaxGroups; ++q) {
    if (ws + 32 * q < we) {
      const int64_t r = ws + 32 * q + lane;
      const bool valid = r < we;
      const uint32_t bb = bk[q] & 0x7fffffffu;
      const unsigned mask = pm[q];
      const int leader = __ffs(mask) - 1;
      int32_t old = 0;
      if (valid && lane == leader) old = atomicAdd(&my[bb], __popc(mask));
      old = __shfl_sync(0xffffffffu, old, leader);
      if (valid) {
        uint32_t *dst = perm + base[bb] + old + __popc(mask & lt);
        const uint32_t v = (uint32_t)r | (bk[q] & 0x80000000u);
        if (keep)
          asm volatile("st.global.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(dst), "r"(v), "l"(pol) : "memory");
        else
          *dst = v;
      }
    }
  }
}

__global__ void __launch_bounds__(kScatterWarps * 32) cs_scatter_kernel(
    int64_t n, int64_t chunk, int64_t nchunks, uint32_t m, uint64_t key, int64_t row_offset, uint32_t jb,
    uint32_t sb, const int32_t *__restrict__ hist, const int32_t *__restrict__ tile_sums, uint32_t *__restrict__ perm,
    int keep) {
  for (int64_t cb = blockIdx.x; cb < nchunks; cb += gridDim.x) {
    cs_scatter_chunk(cb, n, chunk, nchunks, m, key, row_offset, jb, sb, hist, tile_sums, perm, keep);
    __syncthreads();
  }
}
}  // namespace

cudaError_t launch_hash_export(uint64_t key, uint32_t s, uint32_t M, int64_t row_begin, int64_t count,
                               int32_t *bucket, int8_t *sign, cudaStream_t st, LaunchCounter lc) {
  if (count <= 0) return cudaSuccess;
  int64_t total = count * s;
  int grid = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
  hash_export_kernel<<<grid, 256, 0, st>>>(key, s, M, row_begin, count, bucket, sign);
  lc.add();
  return cudaGetLastError();
}

bool cs_sort_supported(int64_t m) { return m >= 1 && m * (4 + 4 * kScatterWarps) <= 200 * 1024; }

CsSortPlan cs_sort_plan(int64_t n, int64_t m) {
  CsSortPlan p;
  p.n = n;
  p.m = m;
  // ~8 chunks per SM, a multiple of 8 warps x 32 rows, at most 32768 rows (uint16
  // per-warp prefixes), and at most 4M histogram entries.
  int64_t chunk = (n + 148 * 8 - 1) / (148 * 8);
  chunk = std::max<int64_t>(chunk, 1024);
  while (((n + chunk - 1) / chunk) * m > (int64_t(4) << 20) && chunk < 32768) chunk *= 2;
  chunk = (chunk + 255) / 256 * 256;
  chunk = std::min<int64_t>(chunk, (int64_t)kScatterWarps * 32 * 16);  // <= 16 groups of 32 rows per warp
  p.chunk = chunk;
  p.nchunks = std::max<int64_t>(1, (n + chunk - 1) / chunk);
  p.entries = m * p.nchunks;
  p.ntiles = (p.entries + kScanTile - 1) / kScanTile;
  return p;
}

// perm stores carry an L2 evict_last hint: a sector
// of perm is written by ~2 CTAs in 4-byte pieces; kept in L2 it is completed
// there (and read there by the next gather) instead of partially written back
constexpr int keep_env = 1;

cudaError_t launch_cs_sort(const CsSortPlan &p, uint64_t key, int64_t row_offset, uint32_t jb, uint32_t sb, int32_t *hist,
                           int32_t *tile_sums, uint32_t *perm, cudaStream_t st, LaunchCounter lc) {
  const uint32_t m = (uint32_t)p.m;
  size_t hsmem = 4 * (size_t)m;
  IHS_SMEM_ATTR(cs_hist_kernel, hsmem);
  const unsigned grid = (unsigned)p.nchunks;
  cs_hist_kernel<<<grid, kHistThreads, hsmem, st>>>(p.n, p.chunk, p.nchunks, m, key, row_offset, jb, sb,
                                                                    hist);
  scan_tiles_kernel<<<(unsigned)p.ntiles, 1024, 0, st>>>(hist, p.entries, tile_sums);
  scan_sums_kernel<<<1, 1024, 0, st>>>(tile_sums, p.ntiles);
  size_t ssmem = (4 + 4 * kScatterWarps) * (size_t)m;
  IHS_SMEM_ATTR(cs_scatter_kernel, ssmem);
  if (p.n > 0)
    cs_scatter_kernel<<<grid, kScatterWarps * 32, ssmem, st>>>(p.n, p.chunk, p.nchunks, m, key,
                                                                              row_offset, jb, sb, hist, tile_sums, perm,
                                                                              keep_env);
  lc.add(p.n > 0 ? 4 : 3);
  return cudaGetLastError();
}

}  // namespace ihs
