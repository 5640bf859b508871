// Shared device helpers for the sm_100a IHS kernels (product path only; the
// oracle under oracle/ shares nothing with this file).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ihs {

constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;

// splitmix64 step (reading R1): golden-gamma add + finaliser.
__host__ __device__ __forceinline__ uint64_t sm64(uint64_t x) {
  x += kGamma;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// k_t = SM(SM(seed) ^ t): one key per IHS iteration, computed on the host.
__host__ __device__ __forceinline__ uint64_t iter_key(uint64_t seed, uint64_t t) {
  return sm64(sm64(seed) ^ t);
}

// Bucket (within [0, m)) and sign bit of global row gi in SJLT block j.
// bucket = j*M + hi32(hi32(w) * M);  neg = bit 0 of w.
__device__ __forceinline__ uint32_t hash_bucket(uint64_t key, uint64_t gi, uint32_t j, uint32_t s,
                                                uint32_t M, bool &neg) {
  uint64_t w = sm64(key ^ (gi * (uint64_t)s + (uint64_t)j));
  neg = (w & 1ull) != 0;
  return j * M + __umulhi((uint32_t)(w >> 32), M);
}

__device__ __forceinline__ double ldg_stream(const double *p) {
  double v;
  asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Lanes of the warp whose key equals this lane's key (a match_any built from
// one ballot per key bit: MATCH.ANY is a long-latency instruction on sm_100a).
// key < 2^nbits; lanes with valid == false form their own group.
__device__ __forceinline__ unsigned peers_by_ballot(uint32_t key, int nbits, bool valid) {
  const unsigned vm = __ballot_sync(0xffffffffu, valid);
  unsigned peers = valid ? vm : ~vm;
#pragma unroll 4
  for (int k = 0; k < nbits; ++k) {
    const unsigned bk = __ballot_sync(0xffffffffu, (key >> k) & 1u);
    peers &= ((key >> k) & 1u) ? bk : ~bk;
  }
  return peers;
}

// peers_by_ballot with the key width fixed at compile time: the ballots
// unroll into VOTE + select pairs with no per-bit loop or divergence checks
// (sjlt_lists_kernel's placement pass, M = 512: NB = 9).
template <int NB>
__device__ __forceinline__ unsigned peers_by_ballot_c(uint32_t key, bool valid) {
  const unsigned vm = __ballot_sync(0xffffffffu, valid);
  unsigned peers = valid ? vm : ~vm;
#pragma unroll
  for (int k = 0; k < NB; ++k) {
    const bool bit = ((key >> k) & 1u) != 0;
    const unsigned bk = __ballot_sync(0xffffffffu, bit);
    peers &= bit ? bk : ~bk;
  }
  return peers;
}

// Transpose-reduce U per-lane partial sums (one per row) across the warp in
// U-1 + log2(32/U) shuffles instead of U*5.  On return p[0] holds the full sum
// for row reduced_row_of_lane<U>(lane).
template <int U>
__device__ __forceinline__ void transpose_reduce(double (&p)[U], int lane) {
  static_assert(U == 1 || U == 2 || U == 4 || U == 8 || U == 16 || U == 32, "U");
  int sh = 16;
#pragma unroll
  for (int w = U / 2; w >= 1; w >>= 1, sh >>= 1) {
    const bool upper = (lane & sh) != 0;
#pragma unroll
    for (int i = 0; i < w; ++i) {
      double send = upper ? p[i] : p[i + w];
      double keep = upper ? p[i + w] : p[i];
      p[i] = keep + __shfl_xor_sync(0xffffffffu, send, sh);
    }
  }
#pragma unroll
  for (; sh >= 1; sh >>= 1) p[0] += __shfl_xor_sync(0xffffffffu, p[0], sh);
}

template <int U>
__device__ __forceinline__ int reduced_row_of_lane(int lane) {
  int u = 0, sh = 16;
#pragma unroll
  for (int w = U / 2; w >= 1; w >>= 1, sh >>= 1) u += (lane & sh) ? w : 0;
  return u;
}

template <int U>
__device__ __forceinline__ int owner_lane_of_row(int u) {
  int lane = 0, sh = 16;
#pragma unroll
  for (int w = U / 2; w >= 1; w >>= 1, sh >>= 1)
    if (u & w) lane |= sh;
  return lane;
}

// Cholesky pivot: r = 1/sqrt(piv) (one MUFU.RSQ64H + Newton, <= 1 ulp) and
// L_jj = piv * r, instead of an IEEE sqrt followed by an IEEE division: both
// sit on the factorisation's sequential critical path.
__device__ __forceinline__ void pivot_rsqrt(double piv, double &ljj, double &r) {
  r = rsqrt(piv);
  ljj = piv * r;
}

// Device-side status word (first error wins).
__device__ __forceinline__ void set_status(int *status, int code) {
  if (status) atomicCAS(status, 0, code);
}

// Latency-bound single-CTA / single-cluster kernels (the inner solves) ask for
// this much dynamic shared memory so that no other CTA can share their SM:
// the next iteration's sort, prefetched on a side stream, would otherwise
// co-reside and steal issue slots on the critical path.
constexpr size_t kExclusiveSmem = 200 * 1024;

// Opt a kernel into large dynamic shared memory once per call site and size
// (raised only when a launch needs more): cudaFuncSetAttribute must not run on
// every launch.
#define IHS_SMEM_ATTR(func, bytes)                                                                   \
  do {                                                                                               \
    static size_t _ihs_attr_cur = 48 * 1024;                                                         \
    if ((size_t)(bytes) > _ihs_attr_cur) {                                                           \
      cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(bytes));         \
      _ihs_attr_cur = (size_t)(bytes);                                                               \
    }                                                                                                \
  } while (0)

// Copy cnt contiguous doubles global -> shared with 16 loads in flight per
// thread (a runtime-bounded copy loop issues one L2 round trip at a time).
__device__ __forceinline__ void load_rows(double *dst, const double *__restrict__ src, int64_t cnt, int tid,
                                          int nthreads) {
  for (int64_t e0 = tid; e0 < cnt; e0 += 16 * (int64_t)nthreads) {
    double v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int64_t e = e0 + (int64_t)k * nthreads;
      v[k] = e < cnt ? src[e] : 0.0;
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int64_t e = e0 + (int64_t)k * nthreads;
      if (e < cnt) dst[e] = v[k];
    }
  }
}

}  // namespace ihs
