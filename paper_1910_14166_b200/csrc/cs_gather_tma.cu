// a2 (+ a5 fused) for dense CountSketch, TMA-fed: one CTA per bucket.  A
// producer warp streams the bucket's rows (ascending, from the stable sort)
// into a shared-memory ring (~24 KiB in flight per CTA) with 1-D bulk copies (cp.async.bulk -> UBLKCP), one per
// row, completing on an mbarrier per stage.  Each thread owns one column: it
// adds sign*A[row, c] for the rows of a stage in ring order, i.e. the same
// left-to-right fp64 sum as the oracle (SA bit-identical at P = 1).  With the
// gradient fused, each warp first reduces the dot products a_i.x of its rows
// of the stage (r_i = b_i - a_i.x to shared memory), then every thread also
// accumulates g_c += r_i A[i, c].  A is read from HBM once per iteration.
//
// PAPER.md:236-240 (stream A; bucket h(i) accumulates +-row i) and Eq. (2),
// PAPER.md:83-86 (the linear term A^T(b - A x^t)).
#include "common.cuh"
#include "kernels.h"

#include <cstdlib>
#include <type_traits>

namespace ihs {

namespace {
constexpr int kScanTile = 4096;
constexpr int kMaxStages = 8;
constexpr int kRingBytes = 24 * 1024;  // bytes in flight per CTA (~168 KiB per SM at 7 CTAs)
constexpr int kDefaultRows = 4;  // rows per stage
constexpr int kDefaultCW = 2;    // consumer warps

__device__ __forceinline__ int32_t scanned_at(const int32_t *hist, const int32_t *tile_sums, int64_t e) {
  return hist[e] + tile_sums[e / kScanTile];
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
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
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// The same copy with an L2 eviction-priority hint (evict_first for A: the
// stream does not push the sort arrays and b out of L2).
__device__ __forceinline__ void bulk_g2s_hint(void *dst, const void *src, uint32_t bytes, uint64_t *bar,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Warps 0-1 consume: thread t owns columns t + 64 q (q < NC) of the bucket's
// SA row and gradient partial; it reads the stage's rows from shared memory in
// ring order, so every column is a left-to-right sum.  With the gradient fused,
// each warp transpose-reduces its partial dot products of the stage's 8 rows,
// the two warp partials meet in shared memory behind a named barrier, and every
// thread forms the same residual r_i = b_i - (p0 + p1).  Warp 2 produces: it
// holds the perm entries and b values a window ahead, waits until the slot
// is released (one arrival per consumer warp) and issues one bulk copy per row.
template <bool FUSE, int NC, bool SOLO, int CW, int KR>
__global__ void __launch_bounds__(32 * CW + 32, NC * KR * CW >= 32 ? 6 : 7) cs_gather_tma_kernel(
    const double *__restrict__ A, int64_t n, int d, int m, const int32_t *__restrict__ hist,
    const int32_t *__restrict__ tile_sums, int64_t nchunks, const uint32_t *__restrict__ perm,
    const double *__restrict__ bvec, const double *__restrict__ x, double *__restrict__ SA,
    double *__restrict__ gpart, double scale, int kStages, GatherBatchStrides bst) {
  constexpr int KC = 32 * CW;  // consumer threads
  extern __shared__ __align__(128) unsigned char smem_raw[];
  // blockIdx.y selects one SJLT block of a batch (its own sort and SA rows);
  // the gradient rides on batch entry 0 only
  hist += blockIdx.y * bst.hist;
  tile_sums += blockIdx.y * bst.tiles;
  perm += blockIdx.y * bst.perm;
  SA += blockIdx.y * bst.sa;
  const bool fz = FUSE && (SOLO || blockIdx.y == 0);  // SOLO: a one-entry batch (compile-time)
  double *ring = reinterpret_cast<double *>(smem_raw);                                // [kStages][KR][d]
  double *bs = ring + (size_t)kStages * KR * d;                                    // [kStages][KR]
  double *pd = bs + kStages * KR;                                                  // [kStages][CW][KR]
  uint64_t *full = reinterpret_cast<uint64_t *>(pd + kStages * CW * KR);          // [kStages]
  uint64_t *empty = full + kMaxStages;                                                // [kStages]
  double *sgn = reinterpret_cast<double *>(empty + kMaxStages);                       // [kStages][KR] +-1
  const int b = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int64_t beg = scanned_at(hist, tile_sums, (int64_t)b * nchunks);
  int64_t end = (b + 1 < m) ? scanned_at(hist, tile_sums, (int64_t)(b + 1) * nchunks) : n;
  if (gridDim.z > 1) {
    // few buckets: segment z of the bucket's (ascending) rows -> partial sums
    // in SA + z * bst.seg_sa / gpart + z * m * d, summed in segment order after
    const int64_t L = end - beg, z = blockIdx.z, nz = gridDim.z;
    end = beg + L * (z + 1) / nz;
    beg = beg + L * z / nz;
    SA += z * bst.seg_sa;
    if (gpart) gpart += z * (int64_t)m * d;
  }
  const int64_t len = end - beg;
  const int64_t nb = (len + KR - 1) / KR;
  const uint32_t row_bytes = (uint32_t)d * 8u;

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == CW) {
    // ---------------- producer warp
    // The bucket's perm entries (and, fused, the b values they index) are
    // loaded a 32-row window at a time, one entry per lane, two windows ahead
    // for perm and one ahead for b (whose address depends on perm): neither
    // dependent load sits on the per-stage path.  Each stage takes its KR
    // entries from the current window by shuffle.
    constexpr int kWinStages = 32 / KR;
    const int64_t nwin = (len + 31) / 32;
    auto perm_win = [&](int64_t w) -> uint32_t {
      const int64_t i = w * 32 + lane;
      return (w < nwin && i < len) ? perm[beg + i] : 0u;
    };
    auto b_win = [&](int64_t w, uint32_t e) -> double {
      return (fz && w < nwin && w * 32 + lane < len) ? bvec[e & 0x7fffffffu] : 0.0;
    };
    uint64_t pol = 0;
    if (bst.hint) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    uint32_t p_cur = perm_win(0), p_next = perm_win(1);
    int s = 0;
    uint32_t ph = 0;
    double b_cur = b_win(0, p_cur);
    for (int64_t w = 0; w < nwin; ++w) {
      const uint32_t p_nn = perm_win(w + 2);
      const double b_next = b_win(w + 1, p_next);
#pragma unroll 1
      for (int ks = 0; ks < kWinStages; ++ks) {
        const int64_t k = w * kWinStages + ks;
        if (k >= nb) break;
        const int cnt = (int)min((int64_t)KR, len - k * KR);
        const int src = ks * KR + (lane & (KR - 1));
        const uint32_t e = __shfl_sync(0xffffffffu, p_cur, src);
        const double bv = fz ? __shfl_sync(0xffffffffu, b_cur, src) : 0.0;
        if (k >= kStages) mbar_wait(&empty[s], ph ^ 1u);
        if (lane < cnt) {
          sgn[s * KR + lane] = (e >> 31) ? -1.0 : 1.0;
          if (fz) bs[s * KR + lane] = bv;
        }
        __syncwarp();
        if (lane == 0) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_expect_tx(&full[s], (uint32_t)cnt * row_bytes);
        }
        __syncwarp();
        if (lane < cnt) {
          if (bst.hint)
            bulk_g2s_hint(ring + ((size_t)s * KR + lane) * d, A + (int64_t)(e & 0x7fffffffu) * d, row_bytes,
                          &full[s], pol);
          else
            bulk_g2s(ring + ((size_t)s * KR + lane) * d, A + (int64_t)(e & 0x7fffffffu) * d, row_bytes, &full[s]);
        }
        if (++s == kStages) {
          s = 0;
          ph ^= 1u;
        }
      }
      p_cur = p_next;
      b_cur = b_next;
      p_next = p_nn;
    }
    return;
  }
  // ---------------- consumer warps
  int cc[NC];
  bool cv[NC];
  double acc[NC], gac[NC], xv[NC];
#pragma unroll
  for (int q = 0; q < NC; ++q) {
    const int c = tid + KC * q;
    cv[q] = c < d;
    cc[q] = cv[q] ? c : d - 1;
    acc[q] = 0.0;
    gac[q] = 0.0;
    xv[q] = (fz && cv[q]) ? x[c] : 0.0;
  }
  const int myu = reduced_row_of_lane<KR>(lane);
  const bool owner = owner_lane_of_row<KR>(myu) == lane;
  // loop-invariant shared-memory offsets of this thread's columns in a stage
  int off[KR][NC];
#pragma unroll
  for (int r = 0; r < KR; ++r)
#pragma unroll
    for (int q = 0; q < NC; ++q) off[r][q] = r * d + cc[q];
  int s = 0;
  uint32_t ph = 0;
  // One stage.  FULL (every stage but a bucket's last): no row predicates, so
  // the stage is straight-line code.  The sign is applied as fma(+-1, a, acc),
  // which rounds exactly like acc + (+-a): the ascending-row sum is unchanged.
  auto stage = [&](auto full_tag, int cnt) {
    constexpr bool FULL = decltype(full_tag)::value;
    const double *st = ring + (size_t)s * KR * d;
    double a[KR][NC];
#pragma unroll
    for (int r = 0; r < KR; ++r)
#pragma unroll
      for (int q = 0; q < NC; ++q) a[r][q] = (FULL || r < cnt) ? st[off[r][q]] : 0.0;
    double res[KR];
#pragma unroll
    for (int r = 0; r < KR; ++r) res[r] = 0.0;
    if (fz) {
      double p[KR];
#pragma unroll
      for (int r = 0; r < KR; ++r) {
        p[r] = a[r][0] * xv[0];
#pragma unroll
        for (int q = 1; q < NC; ++q) p[r] = fma(a[r][q], xv[q], p[r]);
      }
      transpose_reduce<KR>(p, lane);
      if (owner) pd[(s * CW + warp) * KR + myu] = p[0];
      if constexpr (CW > 1) {
        asm volatile("bar.sync 1, %0;" ::"n"(KC) : "memory");
      } else {
        __syncwarp();
      }
#pragma unroll
      for (int r = 0; r < KR; ++r) {
        double dot = pd[(s * CW + 0) * KR + r];
#pragma unroll
        for (int w = 1; w < CW; ++w) dot += pd[(s * CW + w) * KR + r];
        res[r] = (FULL || r < cnt) ? bs[s * KR + r] - dot : 0.0;
      }
    }
#pragma unroll
    for (int r = 0; r < KR; ++r) {
      if (FULL || r < cnt) {
        const double sg = sgn[s * KR + r];
#pragma unroll
        for (int q = 0; q < NC; ++q) {
          acc[q] = fma(sg, a[r][q], acc[q]);
          if (fz) gac[q] = fma(res[r], a[r][q], gac[q]);
        }
      }
    }
  };
  const int64_t nfull = len / KR;
  for (int64_t k = 0; k < nb; ++k) {
    mbar_wait(&full[s], ph);
    if (k < nfull)
      stage(std::true_type{}, KR);
    else
      stage(std::false_type{}, (int)(len - k * KR));
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (++s == kStages) {
      s = 0;
      ph ^= 1u;
    }
  }
#pragma unroll
  for (int q = 0; q < NC; ++q) {
    if (cv[q]) {
      SA[(int64_t)b * d + tid + KC * q] = scale == 1.0 ? acc[q] : acc[q] * scale;
      if (fz) gpart[(int64_t)b * d + tid + KC * q] = gac[q];
    }
  }
}

template <bool FUSE, int NC, int CW, int KR>
void launch_tma_t(size_t smem, int nst, int nb, GatherBatchStrides bst, const double *A, int64_t n, int d, int m,
                  const int32_t *hist, const int32_t *tile_sums, int64_t nchunks, const uint32_t *perm,
                  const double *bvec, const double *x, double *SA, double *gpart, double scale, cudaStream_t st) {
  if (nb == 1) {
    IHS_SMEM_ATTR((cs_gather_tma_kernel<FUSE, NC, true, CW, KR>), smem);
    cs_gather_tma_kernel<FUSE, NC, true, CW, KR><<<dim3((unsigned)m, 1, (unsigned)bst.nseg), 32 * CW + 32, smem, st>>>(
        A, n, d, m, hist, tile_sums, nchunks, perm, bvec, x, SA, gpart, scale, nst, bst);
  } else {
    IHS_SMEM_ATTR((cs_gather_tma_kernel<FUSE, NC, false, CW, KR>), smem);
    cs_gather_tma_kernel<FUSE, NC, false, CW, KR>
        <<<dim3((unsigned)m, (unsigned)nb, (unsigned)bst.nseg), 32 * CW + 32, smem, st>>>(
            A, n, d, m, hist, tile_sums, nchunks, perm, bvec, x, SA, gpart, scale, nst, bst);
  }
}
}  // namespace

bool cs_gather_tma_supported(int64_t d, const void *A) {
  return d >= 2 && d <= 256 && (d % 2) == 0 && (reinterpret_cast<uintptr_t>(A) % 16) == 0;
}

cudaError_t launch_cs_gather_tma(const double *A, int64_t n, int64_t d, int64_t m, const int32_t *hist,
                                 const int32_t *tile_sums, int64_t nchunks, const uint32_t *perm, const double *bvec,
                                 const double *x, double *SA, double *gpart, double scale, cudaStream_t st,
                                 LaunchCounter lc, int nbatch, GatherBatchStrides bst) {
  // A's bulk copies carry an L2 evict_first hint: the 4 GiB stream then leaves
  // the sort arrays, b and the partials in L2 (C2 gather with the next sort
  // beside it 0.746 -> 0.724 ms; 0.714 with the scatter's evict_last perm
  // stores, cs_sort.cu).  Two consumer warps and 4-row stages (one warp and
  // 8-row stages measured slower).
  bst.hint = 1;
  const bool f = gpart != nullptr;
  const int CWv = kDefaultCW;
  const int KRv = kDefaultRows;
  // Bytes of rows in flight per CTA, measured per shape on B200 (step time):
  // the fused single-block gather (C2, d = 128) 16 KiB 0.688 / 24 KiB 0.738 /
  // 12 KiB 0.705 / 20 KiB 0.703 ms; d = 256 (C4) 40 KiB 0.771 / 32 KiB 0.775 /
  // 24 KiB 0.784; SJLT batches (C5, d = 96) 24 KiB 34.6 / 12 KiB 35.6 ms.
  const int64_t ring = d >= 192 ? 40 * 1024 : (f && nbatch == 1 && d <= 128) ? 16 * 1024 : kRingBytes;
  const int nst = (int)std::max<int64_t>(2, std::min<int64_t>(kMaxStages, ring / (KRv * d * 8)));
  const size_t smem = (size_t)nst * KRv * d * 8 + (size_t)nst * KRv * 8 * (1 + CWv) + 2 * kMaxStages * 8 +
                      kMaxStages * KRv * 8 + 64;
  const int nc = (int)((d + 32 * CWv - 1) / (32 * CWv));
#define IHS_TMA(NC, CW, KR)                                                                                        \
  (f ? launch_tma_t<true, NC, CW, KR>(smem, nst, nbatch, bst, A, n, (int)d, (int)m, hist, tile_sums, nchunks, perm, \
                                      bvec, x, SA, gpart, scale, st)                                               \
     : launch_tma_t<false, NC, CW, KR>(smem, nst, nbatch, bst, A, n, (int)d, (int)m, hist, tile_sums, nchunks,     \
                                       perm, nullptr, nullptr, SA, nullptr, scale, st))
#define IHS_TMA_NC(CW, KR)   \
  if (nc <= 1)               \
    IHS_TMA(1, CW, KR);      \
  else if (nc == 2)          \
    IHS_TMA(2, CW, KR);      \
  else if (nc <= 4)          \
    IHS_TMA(4, CW, KR);      \
  else                       \
    IHS_TMA(8, CW, KR);
  IHS_TMA_NC(kDefaultCW, kDefaultRows)
#undef IHS_TMA_NC
#undef IHS_TMA
  lc.add();
  return cudaGetLastError();
}

}  // namespace ihs
