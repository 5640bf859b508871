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
// kR rows and every block, the chunk's rows stably sorted by bucket (u16: the
// row's byte offset in a stage tile | sign << 3) and the bucket offsets.  The sum per bucket runs in ascending
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

// List block of one chunk (u16 elements): for each block j, off[j][0..M]
// (bucket t's rows are ent[j][off[j][t] .. off[j][t+1])) padded to moff_of(M),
// then ent[j][0..kR): the chunk's rows sorted by bucket, ascending within a
// bucket, as tile_offset(row) | sign << 3.
__host__ __device__ constexpr int moff_of(int M) { return (M + 1 + 7) / 8 * 8; }
__host__ __device__ constexpr int list_block_elems(int S, int M) { return S * (moff_of(M) + kR); }

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

// List entries hold the byte offset, within a stage tile, of the 16-byte half
// with columns 0-1 of row r: SWIZZLE_32B puts the half h of row r at h ^ bit 2
// of r, so the offset is 32r + 16 * bit 2 of r, and the other half sits at
// that offset ^ 16.  The sign rides in bit 3 (offsets are 16-byte aligned), so
// the consumer's per-entry work is one mask + add for the address and one
// shift-add for the +-1.0 multiplier (no swizzle arithmetic; 23 -> 14.5
// instructions per entry, C5 sketch pass 22.0 -> 21.2 ms).
__host__ __device__ constexpr uint32_t tile_offset(uint32_t r) { return 32u * r + 16u * ((r >> 2) & 1u); }
static_assert(32 * kR <= 0x10000, "tile offsets must fit 16 bits");

__device__ __forceinline__ void lds_f64x2(uint32_t a, double &x, double &y) {
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(a));
}

// ---------------------------------------------------------------------------
// Lists (a1): one CTA per chunk of kR local rows, warp j sorts the chunk by the
// bucket of block j (the counter hash of reading R1, global row ids).  Pass 1
// hashes each row once (codes kept in shared memory) and counts per bucket;
// the warp scans its M counts; pass 2 places rows 32 at a time in ascending
// order (rank among equal buckets from ballots), so each bucket's entries
// ascend.  Out: the chunk's list block.  (Placement by shared-memory atomics
// plus a per-list sort measured slower: 2.3 vs 1.8 ms for C5; the ballots at
// compile-time key width: 1.84 -> 1.64 ms; two warps per block, each sorting
// half the rows: 1.64, dropped.)
template <int NB>  // key bits (NB = 0: nbits at run time)
__global__ void __launch_bounds__(32 * kSMax) sjlt_lists_kernel(int64_t n, uint64_t key, int64_t row_offset,
                                                               uint32_t s, uint32_t M, int nbits,
                                                               uint16_t *__restrict__ lists) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int moff = moff_of((int)M);
  const int lbe = list_block_elems((int)s, (int)M);
  uint16_t *blk = reinterpret_cast<uint16_t *>(smem_raw);              // [s][moff + kR]
  uint16_t *code = blk + lbe;                                          // [s][kR]: bucket | neg << 15
  int32_t *cnt = reinterpret_cast<int32_t *>(code + (size_t)s * kR);  // [s][M]
  const int lane = threadIdx.x & 31, j = threadIdx.x >> 5;
  const int64_t r0 = (int64_t)blockIdx.x * kR;
  const int valid = (int)min((int64_t)kR, n - r0);
  if (j < (int)s) {
    uint16_t *off = blk + (size_t)j * (moff + kR);
    uint16_t *ent = off + moff;
    uint16_t *cd = code + (size_t)j * kR;
    int32_t *ct = cnt + (size_t)j * M;
    for (uint32_t b = lane; b < M; b += 32) ct[b] = 0;
    __syncwarp();
    for (int r = lane; r < valid; r += 32) {
      bool neg;
      const uint32_t b = hash_bucket(key, (uint64_t)(row_offset + r0 + r), (uint32_t)j, s, M, neg) - (uint32_t)j * M;
      cd[r] = (uint16_t)(b | (neg ? 0x8000u : 0u));
      atomicAdd(&ct[b], 1);
    }
    __syncwarp();
    int carry = 0;  // exclusive scan of ct -> off (u16) and the running bases (in ct)
    for (uint32_t b0 = 0; b0 < M; b0 += 32) {
      const uint32_t b = b0 + lane;
      const int v = b < M ? ct[b] : 0;
      int incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const int ex = carry + incl - v;
      if (b < M) {
        off[b] = (uint16_t)ex;
        ct[b] = ex;
      }
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) off[M] = (uint16_t)carry;
    for (int b = (int)M + 1 + lane; b < moff; b += 32) off[b] = 0;
    __syncwarp();
    for (int rb = 0; rb < valid; rb += 32) {  // stable placement, 32 rows at a time
      const int r = rb + lane;
      const bool v = r < valid;
      const uint32_t c = v ? cd[r] : 0u;
      const uint32_t b = c & 0x7fffu;
      const unsigned peers = NB > 0 ? peers_by_ballot_c<NB>(b, v) : peers_by_ballot(b, nbits, v);
      const int rank = __popc(peers & lanemask_lt());
      int base = 0;
      if (v) base = ct[b];
      __syncwarp();
      if (v) {
        ent[base + rank] = (uint16_t)(tile_offset(r) | ((c >> 12) & 8u));
        if (rank == 0) ct[b] = base + __popc(peers);
      }
      __syncwarp();
    }
    for (int r = valid + lane; r < kR; r += 32) ent[r] = 0;
  }
  __syncthreads();
  const uint4 *src = reinterpret_cast<const uint4 *>(blk);
  uint4 *dst = reinterpret_cast<uint4 *>(lists + (size_t)blockIdx.x * lbe);
  for (int i = threadIdx.x; i < lbe / 8; i += blockDim.x) dst[i] = src[i];
}

// a5 riding on the sketch pass: kGradWarps extra warps per CTA stream whole
// rows of A (coalesced loads that bypass L1) and accumulate g's partial
// r_i a_i, r_i = b_i - a_i x, in registers -- the pass is bound by shared
// memory, these warps by HBM, so the gradient's own read of A (4.3 ms for C5)
// hides under the sketch.  The rows follow the sketch: for every chunk w of
// every item (slice q, group g) the CTA takes, its gradient warps read share q
// of chunk w's rows (rows w kR + [q kR / nslices, (q+1) kR / nslices)), paced
// to at most kGradAhead chunks ahead of the CTA's producer.  The nslices CTAs
// of a group walk its chunks together, so the whole rows the gradient reads
// are, within the L2 window, the lines the slices' TMA boxes fetch (or the
// other way round).  ncu at C5 (sketch + gradient launch): DRAM reads 81.9 GB
// (static row ranges, evict_first boxes) -> 48.6 GB (this; A = 25.8 GB), the
// launch 22.98 -> 22.93 ms (8 rows per warp step: the warps are latency-bound,
// 4 rows measured 25.7 ms once paced).  Every row has one fixed warp
// and position in that warp's order: one partial row per warp in gpart,
// reduced in fixed order afterwards (deterministic).
constexpr int kGradWarps = 3;   // 16 consumer + 1 producer + 3 = 20 warps: 5 per SM sub-partition at 96 registers
constexpr int kGradU = 8;       // rows per warp step (loads in flight: the warps are latency-bound)
constexpr int kGradMaxNV = 4;   // d <= 128 (wider rows: the separate gradient pass)
constexpr int kGradAhead = 4;   // chunks the gradient may read ahead of the producer's TMA issue
template <int NV>
__device__ __forceinline__ void grad_warp(const double *__restrict__ A, int64_t n, int d,
                                          const double *__restrict__ bvec, const double *__restrict__ x,
                                          double *__restrict__ gpart, int wk, int nslices, int ngroups,
                                          int64_t nchunks, const volatile int *issued, int lane) {
  constexpr int U = kGradU;
  int colc[NV];
  double xv[NV], gacc[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const int col = lane + 32 * k;
    colc[k] = col < d ? col : d - 1;  // clamped columns carry x = 0
    xv[k] = col < d ? x[col] : 0.0;
    gacc[k] = 0.0;
  }
  const int nitems = nslices * ngroups;
  int64_t kc = 0;  // the CTA's chunk sequence number (the producer's k)
  for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
    const int g = it / nslices, q = it % nslices;
    const int64_t w0 = nchunks * g / ngroups, w1 = nchunks * (g + 1) / ngroups;
    for (int64_t w = w0; w < w1; ++w, ++kc) {
      if (lane == 0)
        while ((int64_t)*issued < kc - kGradAhead) __nanosleep(200);
      __syncwarp();
      const int64_t r0 = min(n, w * kR + (int64_t)q * kR / nslices);
      const int64_t r1 = min(n, w * kR + (int64_t)(q + 1) * kR / nslices);
#pragma unroll 1
      for (int64_t base = r0 + (int64_t)wk * U; base < r1; base += (int64_t)kGradWarps * U) {
        double v[U][NV];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t row = (base + u < r1) ? base + u : r1 - 1;  // clamped rows carry r = 0
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
    }
  }
  const int64_t gw = (int64_t)blockIdx.x * kGradWarps + wk;
#pragma unroll
  for (int k = 0; k < NV; ++k)
    if (lane + 32 * k < d) gpart[gw * d + lane + 32 * k] = gacc[k];
}

// ---------------------------------------------------------------------------
// Sketch: one CTA per SM.  Work items (slice q of kC columns, row group g) are
// dealt round-robin; an item streams its chunks through a 2-stage ring: the
// producer thread issues kR/256 TMA boxes (kC columns x 256 rows, SWIZZLE_32B,
// A with an L2 evict_first hint) and one bulk copy of the chunk's list block.
// Consumer thread t owns bucket t of every block j < S: acc[j][0..3]; it walks
// block j's list of its bucket.  (Measured alternatives, C5: two entries per
// 4-byte load 23.2 ms; four blocks merged into one list per thread with the
// block selecting the accumulator by a 0/+-1 weight 22.3; this loop 21.6.)
template <int S, int NV>
__global__ void __maxnreg__(96) sjlt_onepass_kernel(
    const __grid_constant__ CUtensorMap tmap, const uint16_t *__restrict__ lists, int64_t n, int d, int M,
    int nslices, int ngroups, int64_t nchunks, double *__restrict__ part, const double *__restrict__ A,
    const double *__restrict__ bvec,
    const double *__restrict__ x, double *__restrict__ gpart) {
  extern __shared__ __align__(1024) unsigned char smem_dyn[];
  // stage buffers 1024-byte aligned (the SWIZZLE_32B pattern is a function of the address)
  unsigned char *smem_raw = smem_dyn + ((1024u - (smem_u32(smem_dyn) & 1023u)) & 1023u);
  const int moff = moff_of(M);
  const int lbe = list_block_elems(S, M);
  const uint32_t lb_bytes = (uint32_t)lbe * 2u;
  // [tile 0][tile 1][lists 0][lists 1][barriers]: the tiles 1024-byte aligned
  unsigned char *tiles = smem_raw;
  unsigned char *lbuf = smem_raw + kStages * kTileBytes;
  uint64_t *full = reinterpret_cast<uint64_t *>(lbuf + kStages * lb_bytes);
  uint64_t *empty = full + kStages;
  int *issued = reinterpret_cast<int *>(empty + kStages);  // chunks whose TMA the producer has issued, minus 1
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumers / 32);
    }
    *issued = -1;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (NV > 0 && warp > kConsumers / 32) {
    grad_warp<NV ? NV : 1>(A, n, d, bvec, x, gpart, warp - kConsumers / 32 - 1, nslices, ngroups, nchunks,
                           issued, lane);
    return;
  }
  const int nitems = nslices * ngroups;
  if (warp == kConsumers / 32) {
    // ---------------- producer
    if (lane == 0) {
      uint64_t pol;
      // evict_normal, not evict_first: the neighbouring slices' CTAs (and the
      // gradient warps) read the rest of every 256-byte line a box promotes,
      // so the sketch takes A from HBM once (ncu, C5 sketch only: 33.2 GB with
      // evict_first, 26.5 GB with evict_normal, A = 25.8 GB; same time)
      asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
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
          *reinterpret_cast<volatile int *>(issued) = (int)k;
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
      if (owner) {
        const uint32_t tb = smem_u32(tiles) + (uint32_t)s * kTileBytes;  // 1024-byte aligned
        const uint16_t *lb = reinterpret_cast<const uint16_t *>(lbuf + (size_t)s * lb_bytes);
#pragma unroll
        for (int j = 0; j < S; ++j) {
          const uint16_t *off = lb + j * (moff + kR);
          const uint16_t *ent = off + moff;
          const int o0 = off[tid], o1 = off[tid + 1];
#pragma unroll 2
          for (int e = o0; e < o1; ++e) {
            const uint32_t en = ent[e];
            const double sg = __hiloint2double((int)((en << 28) + 0x3ff00000u), 0);  // bit 3 -> sign bit
            const uint32_t a = tb + (en & 0xfff0u);
            double x0, x1, x2, x3;
            lds_f64x2(a, x0, x1);
            lds_f64x2(a ^ 16u, x2, x3);
            acc[j][0] = fma(sg, x0, acc[j][0]);
            acc[j][1] = fma(sg, x1, acc[j][1]);
            acc[j][2] = fma(sg, x2, acc[j][2]);
            acc[j][3] = fma(sg, x3, acc[j][3]);
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
  return kStages * ((size_t)kTileBytes + (size_t)list_block_elems(S, M) * 2) + 2 * kStages * 8 + 16 + 1024;
}
size_t lists_smem(int S, int M) { return (size_t)list_block_elems(S, M) * 2 + (size_t)S * kR * 2 + (size_t)S * M * 4; }
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
  const int nbits = p.M > 1 ? 32 - __builtin_clz((unsigned)(p.M - 1)) : 1;
#define IHS_LISTS(NBV)                                                                                        \
  {                                                                                                           \
    IHS_SMEM_ATTR(sjlt_lists_kernel<NBV>, smem);                                                              \
    sjlt_lists_kernel<NBV><<<(unsigned)p.nchunks, 32 * p.s, smem, st>>>(p.n, key, row_offset, (uint32_t)p.s, \
                                                                        (uint32_t)p.M, nbits, lists);         \
  }
  switch (nbits) {
    case 8: IHS_LISTS(8) break;
    case 9: IHS_LISTS(9) break;
    case 10: IHS_LISTS(10) break;
    default: IHS_LISTS(0) break;
  }
#undef IHS_LISTS
  lc.add();
  return cudaGetLastError();
}

int sjlt_onepass_grad_blocks(const SjltOnepassPlan &p) {
  return (p.d + 31) / 32 <= kGradMaxNV ? p.grid * kGradWarps : 0;
}

cudaError_t launch_sjlt_onepass(const SjltOnepassPlan &p, const double *A, const uint16_t *lists, double *partials,
                                double *SA, double scale, cudaStream_t st, LaunchCounter lc, const double *bvec,
                                const double *x, double *gpart) {
  CUtensorMap tm;
  cuuint64_t gdim[2] = {(cuuint64_t)p.d, (cuuint64_t)p.n};
  cuuint64_t gstr[1] = {(cuuint64_t)p.d * 8};
  cuuint32_t box[2] = {(cuuint32_t)kC, (cuuint32_t)kBoxRows};
  cuuint32_t es[2] = {1, 1};
  if (encode_fn()(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double *>(A), gdim, gstr, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  const int nv = gpart ? (int)((p.d + 31) / 32) : 0;
  if (nv > kGradMaxNV) return cudaErrorInvalidValue;
  const unsigned threads = kConsumers + 32 + (nv ? 32 * kGradWarps : 0);
#define IHS_ONEPASS_NV(SV, NVV)                                                                                \
  case NVV:                                                                                                    \
    IHS_SMEM_ATTR((sjlt_onepass_kernel<SV, NVV>), p.smem);                                                     \
    sjlt_onepass_kernel<SV, NVV><<<p.grid, threads, p.smem, st>>>(tm, lists, p.n, (int)p.d, (int)p.M, p.nslices, \
                                                                  p.ngroups, p.nchunks, partials, A, bvec, x,  \
                                                                  gpart);                                        \
    break;
#define IHS_ONEPASS(SV)        \
  case SV:                     \
    switch (nv) {              \
      IHS_ONEPASS_NV(SV, 0)    \
      IHS_ONEPASS_NV(SV, 1)    \
      IHS_ONEPASS_NV(SV, 2)    \
      IHS_ONEPASS_NV(SV, 3)    \
      IHS_ONEPASS_NV(SV, 4)    \
    }                          \
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
#undef IHS_ONEPASS_NV
  lc.add();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return launch_sum_splits(partials, p.m * p.d, p.ngroups, scale, SA, st, lc);
}

}  // namespace ihs
