// a2 for dense SJLT (s > 1) in ONE read of A (section 2: s
// independent CountSketch blocks of m/s rows each, every column of S has s
// nonzeros +-1/sqrt(s); streaming A once, bucket h_j(i) of
// block j accumulates +-row i).
//
// Why this shape: every element of A must meet s
// accumulators.  Fanning rows out to s owner SMs through L2 is capped by the
// L2->SM delivery rate (~8.5 TB/s measured: 8 x 25.8 GB for C5 = 24 ms), TMA
// multicast measured slower still (tools/probe/mc_probe.cu), so each element
// enters exactly ONE SM: the SM that owns ALL m buckets of a 4-column slice.
// Its 512 consumer threads own one bucket of every block (thread t: bucket t of
// blocks 0..s-1) with the 4 columns of each in registers, so a (row, block)
// pair is a register update by its owner thread -- no shared-memory
// read-modify-write, no atomics.  The owner finds its rows through per-chunk
// lists built once per iteration by sjlt_lists_kernel: for every chunk of
// kR rows and every block, the chunk's rows stably sorted by bucket (u16 row |
// sign << 15) and the bucket offsets.  The sum per bucket runs in ascending
// row order inside a chunk, chunks ascending inside a row group; the row-group
// partials are added in group order (deterministic; within rounding of the
// oracle's single left-to-right sum, reading R3).
#include "common.cuh"
#include "kernels.h"

#include <cuda.h>

#include <algorithm>
#include <cstring>

namespace ihs {

namespace {
constexpr int kR = 2048;          // rows per chunk (entries: row in 11 bits)
constexpr int kC = 4;             // columns per slice (32 B per row: the SWIZZLE_32B TMA atom)
constexpr int kBoxRows = 256;     // TMA box rows (box dims <= 256)
constexpr int kSMax = 8;          // blocks handled in registers
constexpr int kMMax = 512;        // buckets per block (one owner thread each)
constexpr int kConsumers = 512;   // consumer threads (16 warps)
constexpr int kStages = 2;
constexpr int kTileBytes = kR * kC * 8;  // 64 KiB
constexpr int kListThreads = 256;

// List block of one chunk (u16 elements).  For each block j a header
// hdr[j][0..M]: bucket t's list starts at pair hdr[j][t] & 0x7fff of block j's
// entry area and holds 2 (hdr[j][t+1] - hdr[j][t]) - (hdr[j][t] >> 15) entries
// (bit 15: the list's last pair is half empty); then the entry areas (cap_of(M)
// entries each), lists padded to whole pairs (one 4-byte load per two
// entries).  Entry = row | sign << 15, rows ascending within a list.
__host__ __device__ constexpr int hpad_of(int M) { return (M + 1 + 7) / 8 * 8; }
__host__ __device__ constexpr int cap_of(int M) { return (kR + M + 7) / 8 * 8; }
__host__ __device__ constexpr int header_elems(int S, int M) { return S * hpad_of(M); }
__host__ __device__ constexpr int area_start(int S, int M, int j) { return header_elems(S, M) + j * cap_of(M); }
__host__ __device__ constexpr int list_block_elems(int S, int M) { return area_start(S, M, S); }

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_box(void *dst, const CUtensorMap *tm, int c0, int c1, uint64_t *bar,
                                        uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
      "%3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(tm), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ---------------------------------------------------------------------------
// Lists (a1): one CTA per chunk of kR local rows.  Every (row, block) pair is
// hashed (reading R1, global row ids) and counted per (block, bucket); after
// the quad offsets, each pair is placed into its bucket's list (shared-memory
// atomics, in no fixed order) and every list is then sorted by row (lists hold
// ~kR/M entries), so each bucket's sum runs in ascending row order within the
// chunk whatever order the atomics took.
__global__ void __launch_bounds__(kListThreads) sjlt_lists_kernel(int64_t n, uint64_t key, int64_t row_offset,
                                                                 int s, int M, uint16_t *__restrict__ lists) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int hp = hpad_of(M);
  const int lbe = list_block_elems(s, M), he = header_elems(s, M);
  uint16_t *blk = reinterpret_cast<uint16_t *>(smem_raw);  // the block: headers + areas
  uint16_t *cnt = blk + lbe;                               // [s][hp]
  uint16_t *fill = cnt + s * hp;                           // [s][hp]
  const int tid = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.x * kR;
  const int valid = (int)min((int64_t)kR, n - r0);
  for (int e = tid; e < 2 * s * hp; e += blockDim.x) cnt[e] = 0;
  __syncthreads();
  // pairs (j, r) with r fastest: consecutive threads hash consecutive rows
  const int npairs = s * valid;
  for (int p = tid; p < npairs; p += blockDim.x) {
    const int j = p / valid, r = p - j * valid;
    bool neg;
    const uint32_t b =
        hash_bucket(key, (uint64_t)(row_offset + r0 + r), (uint32_t)j, (uint32_t)s, (uint32_t)M, neg) - (uint32_t)j * M;
    atomicAdd(reinterpret_cast<unsigned *>(cnt + j * hp + (b & ~1u)), (b & 1u) ? 0x10000u : 1u);
  }
  __syncthreads();
  // pair offsets: warp j scans ceil(cnt/2) over the buckets of block j
  const int lane = tid & 31, warp = tid >> 5;
  for (int j = warp; j < s; j += kListThreads / 32) {
    const uint16_t *c = cnt + j * hp;
    uint16_t *h = blk + j * hp;
    int carry = 0;
    for (int b0 = 0; b0 < M; b0 += 32) {
      const int b = b0 + lane;
      const int v = b < M ? (c[b] + 1) / 2 : 0;
      int incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (b < M) h[b] = (uint16_t)((carry + incl - v) | ((c[b] & 1) ? 0x8000 : 0));
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    for (int b = M + lane; b < hp; b += 32) h[b] = (uint16_t)carry;
  }
  __syncthreads();
  for (int p = tid; p < npairs; p += blockDim.x) {
    const int j = p / valid, r = p - j * valid;
    bool neg;
    const uint32_t b =
        hash_bucket(key, (uint64_t)(row_offset + r0 + r), (uint32_t)j, (uint32_t)s, (uint32_t)M, neg) - (uint32_t)j * M;
    const uint32_t old = atomicAdd(reinterpret_cast<unsigned *>(fill + j * hp + (b & ~1u)), (b & 1u) ? 0x10000u : 1u);
    const uint32_t rank = (b & 1u) ? (old >> 16) : (old & 0xffffu);
    blk[area_start(s, M, j) + 2 * (blk[j * hp + b] & 0x7fff) + rank] = (uint16_t)(r | (neg ? 0x8000 : 0));
  }
  __syncthreads();
  // sort each list by row (insertion sort: a few entries each); pad to pairs
  for (int L = tid; L < s * M; L += blockDim.x) {
    const int j = L / M, t = L - j * M;
    const int nn = cnt[j * hp + t];
    uint16_t *e = blk + area_start(s, M, j) + 2 * (blk[j * hp + t] & 0x7fff);
    for (int i = 1; i < nn; ++i) {
      const uint16_t v = e[i];
      int k = i - 1;
      while (k >= 0 && (e[k] & 0x7fffu) > (v & 0x7fffu)) {
        e[k + 1] = e[k];
        --k;
      }
      e[k + 1] = v;
    }
    if (nn & 1) e[nn] = 0;
  }
  __syncthreads();
  uint4 *g = reinterpret_cast<uint4 *>(lists + (size_t)blockIdx.x * lbe);
  for (int i = tid; i < lbe / 8; i += blockDim.x) g[i] = reinterpret_cast<const uint4 *>(blk)[i];
}

// Row (entry & 0x7fff) of a stage tile, times the entry's sign (bit 15):
// SWIZZLE_32B puts the 16-byte half h of row r at h ^ bit 2 of r; the sign is a
// flip of the doubles' sign bits (exact, like the oracle's +-a).
__device__ __forceinline__ void tile_row(const unsigned char *st, uint32_t e, double2 &lo, double2 &hi) {
  const uint32_t r = e & 0x7fffu;
  const uint32_t sw = (r >> 2) & 1u;
  lo = *reinterpret_cast<const double2 *>(st + r * 32u + 16u * sw);
  hi = *reinterpret_cast<const double2 *>(st + r * 32u + 16u * (sw ^ 1u));
  const uint32_t flip = (e & 0x8000u) << 16;
  lo.x = __hiloint2double(__double2hiint(lo.x) ^ (int)flip, __double2loint(lo.x));
  lo.y = __hiloint2double(__double2hiint(lo.y) ^ (int)flip, __double2loint(lo.y));
  hi.x = __hiloint2double(__double2hiint(hi.x) ^ (int)flip, __double2loint(hi.x));
  hi.y = __hiloint2double(__double2hiint(hi.y) ^ (int)flip, __double2loint(hi.y));
}

// ---------------------------------------------------------------------------
// Sketch: one CTA per SM.  Work items (slice q of kC columns, row group g) are
// dealt round-robin; an item streams its chunks through a 2-stage ring: the
// producer thread issues kR/256 TMA boxes (kC columns x 256 rows, SWIZZLE_32B,
// A with an L2 evict_first hint) and one bulk copy of the chunk's list block.
// Consumer thread t owns bucket t of every block j < S: acc[j][0..3]; it walks
// block j's list of its bucket, two entries per 4-byte load.
template <int S>
__global__ void __maxnreg__(96) sjlt_onepass_kernel(
    const __grid_constant__ CUtensorMap tmap, const uint16_t *__restrict__ lists, int64_t n, int d, int M,
    int nslices, int ngroups, int64_t nchunks, double *__restrict__ part) {
  extern __shared__ __align__(1024) unsigned char smem_dyn[];
  // stage buffers 1024-byte aligned (the SWIZZLE_32B pattern is a function of the address)
  unsigned char *smem_raw = smem_dyn + ((1024u - (smem_u32(smem_dyn) & 1023u)) & 1023u);
  const int hp = hpad_of(M);
  const int lbe = list_block_elems(S, M);
  const uint32_t lb_bytes = (uint32_t)lbe * 2u;
  // [tile 0][tile 1][lists 0][lists 1][barriers]: the tiles 1024-byte aligned
  unsigned char *tiles = smem_raw;
  unsigned char *lbuf = smem_raw + kStages * kTileBytes;
  uint64_t *full = reinterpret_cast<uint64_t *>(lbuf + kStages * lb_bytes);
  uint64_t *empty = full + kStages;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumers / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int nitems = nslices * ngroups;
  if (warp == kConsumers / 32) {
    // ---------------- producer
    if (lane == 0) {
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap) : "memory");
      int s = 0;
      uint32_t ph = 0;
      int64_t k = 0;
      for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
        const int g = it / nslices, q = it % nslices;
        const int64_t w0 = nchunks * g / ngroups, w1 = nchunks * (g + 1) / ngroups;
        for (int64_t w = w0; w < w1; ++w, ++k) {
          if (k >= kStages) mbar_wait(&empty[s], ph ^ 1u);
          unsigned char *st = tiles + (size_t)s * kTileBytes;
          mbar_expect_tx(&full[s], (uint32_t)kTileBytes + lb_bytes);
#pragma unroll 1
          for (int bx = 0; bx < kR / kBoxRows; ++bx)
            tma_box(st + bx * kBoxRows * kC * 8, &tmap, q * kC, (int)(w * kR + bx * kBoxRows), &full[s], pol);
          bulk_g2s(lbuf + (size_t)s * lb_bytes, lists + (size_t)w * lbe, lb_bytes, &full[s]);
          if (++s == kStages) {
            s = 0;
            ph ^= 1u;
          }
        }
      }
    }
    return;
  }
  // ---------------- consumers
  const bool owner = tid < M;
  int s = 0;
  uint32_t ph = 0;
  for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
    const int g = it / nslices, q = it % nslices;
    const int64_t w0 = nchunks * g / ngroups, w1 = nchunks * (g + 1) / ngroups;
    double acc[S][kC];
#pragma unroll
    for (int j = 0; j < S; ++j)
#pragma unroll
      for (int c = 0; c < kC; ++c) acc[j][c] = 0.0;
    for (int64_t w = w0; w < w1; ++w) {
      mbar_wait(&full[s], ph);
      const unsigned char *st = tiles + (size_t)s * kTileBytes;
      const uint16_t *lb = reinterpret_cast<const uint16_t *>(lbuf + (size_t)s * lb_bytes);
      if (owner) {
#pragma unroll
        for (int j = 0; j < S; ++j) {
          const uint32_t h0 = lb[j * hp + tid], h1 = lb[j * hp + tid + 1];
          const uint32_t p0 = h0 & 0x7fffu;
          const int nn = 2 * (int)((h1 & 0x7fffu) - p0) - (int)(h0 >> 15);
          const uint32_t *pairs = reinterpret_cast<const uint32_t *>(lb + area_start(S, M, j)) + p0;
          const int np = nn >> 1;
          uint32_t pr = nn > 0 ? pairs[0] : 0u;
          // two entries per step, the next pair loaded ahead; the two rows are
          // added first (their signs applied as sign-bit flips) and then to the
          // accumulator: one dependent add per pair
#pragma unroll 1
          for (int i = 0; i < np; ++i) {
            const uint32_t nx = (2 * (i + 1) < nn) ? pairs[i + 1] : 0u;
            double2 lo0, hi0, lo1, hi1;
            tile_row(st, pr & 0xffffu, lo0, hi0);
            tile_row(st, pr >> 16, lo1, hi1);
            acc[j][0] += lo0.x + lo1.x;
            acc[j][1] += lo0.y + lo1.y;
            acc[j][2] += hi0.x + hi1.x;
            acc[j][3] += hi0.y + hi1.y;
            pr = nx;
          }
          if (nn & 1) {
            double2 lo0, hi0;
            tile_row(st, pr & 0xffffu, lo0, hi0);
            acc[j][0] += lo0.x;
            acc[j][1] += lo0.y;
            acc[j][2] += hi0.x;
            acc[j][3] += hi0.y;
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++s == kStages) {
        s = 0;
        ph ^= 1u;
      }
    }
    if (owner) {
      double *pg = part + (size_t)g * ((size_t)M * S) * d;
#pragma unroll
      for (int j = 0; j < S; ++j) {
        double *row = pg + ((size_t)j * M + tid) * d + q * kC;
#pragma unroll
        for (int c = 0; c < kC; ++c)
          if (q * kC + c < d) row[c] = acc[j][c];
      }
    }
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      p = nullptr;
    }
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

size_t onepass_smem(int S, int M) {
  return kStages * ((size_t)kTileBytes + (size_t)list_block_elems(S, M) * 2) + 2 * kStages * 8 + 1024;
}
size_t lists_smem(int S, int M) { return ((size_t)list_block_elems(S, M) + (size_t)2 * S * hpad_of(M)) * 2; }
}  // namespace

bool sjlt_onepass_plan(int64_t n, int64_t d, int64_t m, int s, int num_sms, const void *A, SjltOnepassPlan &p) {
  if (s < 2 || s > kSMax || m % s != 0) return false;
  const int64_t M = m / s;
  if (M < 1 || M > kMMax || n < 1 || n > (int64_t(1) << 31) - kR) return false;
  if (d < 2 || (d % 2) != 0 || (reinterpret_cast<uintptr_t>(A) % 16) != 0 || !encode_fn()) return false;
  p = SjltOnepassPlan();
  p.n = n;
  p.d = d;
  p.m = m;
  p.s = s;
  p.M = M;
  p.nchunks = (n + kR - 1) / kR;
  p.nslices = (int)((d + kC - 1) / kC);
  // row groups: items = nslices x ngroups dealt to one CTA per SM; ngroups so
  // that the items divide evenly over the SMs (lcm), at most one chunk per group
  const int64_t gcd = std::__gcd<int64_t>(p.nslices, num_sms);
  p.ngroups = (int)std::max<int64_t>(1, std::min<int64_t>(num_sms / gcd, p.nchunks));
  p.grid = (int)std::min<int64_t>(num_sms, (int64_t)p.nslices * p.ngroups);
  p.lists_bytes = (size_t)p.nchunks * list_block_elems(s, (int)M) * 2;
  p.partial_bytes = (size_t)p.ngroups * m * d * 8;
  p.smem = onepass_smem(s, (int)M);
  return p.smem <= 227 * 1024;
}

cudaError_t launch_sjlt_lists(const SjltOnepassPlan &p, uint64_t key, int64_t row_offset, uint16_t *lists,
                              cudaStream_t st, LaunchCounter lc) {
  const size_t smem = lists_smem(p.s, (int)p.M);
  IHS_SMEM_ATTR(sjlt_lists_kernel, smem);
  sjlt_lists_kernel<<<(unsigned)p.nchunks, kListThreads, smem, st>>>(p.n, key, row_offset, p.s, (int)p.M, lists);
  lc.add();
  return cudaGetLastError();
}

cudaError_t launch_sjlt_onepass(const SjltOnepassPlan &p, const double *A, const uint16_t *lists, double *partials,
                                double *SA, double scale, cudaStream_t st, LaunchCounter lc) {
  CUtensorMap tm;
  cuuint64_t gdim[2] = {(cuuint64_t)p.d, (cuuint64_t)p.n};
  cuuint64_t gstr[1] = {(cuuint64_t)p.d * 8};
  cuuint32_t box[2] = {(cuuint32_t)kC, (cuuint32_t)kBoxRows};
  cuuint32_t es[2] = {1, 1};
  if (encode_fn()(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double *>(A), gdim, gstr, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
#define IHS_ONEPASS(SV)                                                                                            \
  case SV:                                                                                                         \
    IHS_SMEM_ATTR(sjlt_onepass_kernel<SV>, p.smem);                                                                \
    sjlt_onepass_kernel<SV><<<p.grid, kConsumers + 32, p.smem, st>>>(tm, lists, p.n, (int)p.d, (int)p.M,         \
                                                                     p.nslices, p.ngroups, p.nchunks, partials); \
    break;
  switch (p.s) {
    IHS_ONEPASS(2)
    IHS_ONEPASS(3)
    IHS_ONEPASS(4)
    IHS_ONEPASS(5)
    IHS_ONEPASS(6)
    IHS_ONEPASS(7)
    IHS_ONEPASS(8)
    default:
      return cudaErrorInvalidValue;
  }
#undef IHS_ONEPASS
  lc.add();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return launch_sum_splits(partials, p.m * p.d, p.ngroups, scale, SA, st, lc);
}

}  // namespace ihs
