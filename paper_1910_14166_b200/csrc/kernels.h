// Host-side launchers of the sm_100a kernels (internal to libihs.so).
#pragma once
#include <algorithm>
#include <cstdint>
#include <cuda_runtime.h>

namespace ihs {

struct LaunchCounter {
  int64_t *count = nullptr;
  void add(int64_t k = 1) const { if (count) *count += k; }
};

// ---- a1: hash export --------------------------------------------------------
cudaError_t launch_hash_export(uint64_t key, uint32_t s, uint32_t M, int64_t row_begin, int64_t count,
                               int32_t *bucket, int8_t *sign, cudaStream_t st, LaunchCounter lc);

// ---- a1 + a2 (s = 1 dense): stable counting sort of local rows by bucket ----
struct CsSortPlan {
  int64_t n = 0;          // local rows
  int64_t m = 0;          // buckets
  int64_t chunk = 0;      // rows per CTA chunk
  int64_t nchunks = 0;
  int64_t entries = 0;    // m * nchunks
  int64_t ntiles = 0;     // scan tiles
  size_t hist_bytes() const { return (size_t)(entries + 1) * 4; }
  size_t tiles_bytes() const { return (size_t)(ntiles + 1) * 4; }
  size_t perm_bytes() const { return (size_t)n * 4; }
};
CsSortPlan cs_sort_plan(int64_t n, int64_t m);
bool cs_sort_supported(int64_t m);
// hist: entries+1 int32 (bucket-major offsets after the scan); perm: n int32
// (local row | sign << 31), rows of bucket b at [hist[b*nchunks], hist[(b+1)*nchunks]).
// Sorts by the bucket of SJLT block jb of sb (bucket - jb*m in [0, m)); CountSketch: jb = 0, sb = 1.
cudaError_t launch_cs_sort(const CsSortPlan &p, uint64_t key, int64_t row_offset, uint32_t jb, uint32_t sb,
                           int32_t *hist, int32_t *tile_sums, uint32_t *perm, cudaStream_t st, LaunchCounter lc);

// ---- a2 (+a5 fused): bucket-ordered segmented signed row sums ---------------
// SA[b, :] = sum over rows of bucket b (ascending) of sign * A[row, :], times scale.
// If b_vec/x/gpart are non-null: gpart[b, :] = sum_rows A[row,:] * (b_row - A[row,:].x).
cudaError_t launch_cs_gather(const double *A, int64_t n, int64_t d, int64_t m, const int32_t *hist,
                             const int32_t *tile_sums, int64_t nchunks, const uint32_t *perm, const double *bvec,
                             const double *x, double *SA, double *gpart, double scale, cudaStream_t st,
                             LaunchCounter lc);

// TMA-fed variant: one CTA per bucket, bulk copies of whole rows into a smem
// ring.  Requires even d <= 256 and a 16-byte aligned A.  A batch of nbatch
// SJLT blocks runs in one launch (grid.y): entry y uses hist + y*bst.hist,
// tile_sums + y*bst.tiles, perm + y*bst.perm and SA + y*bst.sa; the fused
// gradient (gpart != null) rides on entry 0.
struct GatherBatchStrides {
  int64_t hist = 0, tiles = 0, perm = 0, sa = 0;
  // nseg > 1 (few buckets, long rows lists): grid.z splits every bucket's rows
  // into nseg contiguous segments; segment z writes SA + z * seg_sa and
  // gpart + z * m * d (partials, reduced by the caller in segment order).
  int nseg = 1;
  int64_t seg_sa = 0;
  int hint = 0;  // 1: A's bulk copies carry an L2 evict_first hint
};
bool cs_gather_tma_supported(int64_t d, const void *A);
cudaError_t launch_cs_gather_tma(const double *A, int64_t n, int64_t d, int64_t m, const int32_t *hist,
                                 const int32_t *tile_sums, int64_t nchunks, const uint32_t *perm, const double *bvec,
                                 const double *x, double *SA, double *gpart, double scale, cudaStream_t st,
                                 LaunchCounter lc, int nbatch = 1, GatherBatchStrides bst = GatherBatchStrides());

// ---- a2 dense SJLT (s > 1): smem-tile accumulation --------------------------
struct SjltPlan {
  int64_t n = 0, d = 0, m = 0;
  int s = 0;
  int dc = 0;       // columns per CTA tile
  int nslices = 0;  // ceil(d / dc)
  int nsplit = 0;   // row splits (partials reduced in fixed order)
  size_t smem = 0;
  size_t partial_bytes() const { return (size_t)nsplit * m * d * 8; }
};
bool sjlt_plan(int64_t n, int64_t d, int64_t m, int s, int num_sms, SjltPlan &p);
cudaError_t launch_sjlt_dense(const SjltPlan &p, const double *A, uint64_t key, int64_t row_offset,
                              double *partials, double *SA, double scale, cudaStream_t st, LaunchCounter lc);
// One-read SJLT (2 <= s <= 8, m / s <= 512, even d, 16-byte aligned A;
// sjlt_onepass.cu): per-chunk bucket lists (a1, hashed once per iteration),
// then one pass of column-slice CTAs with register accumulators.
struct SjltOnepassPlan {
  int64_t n = 0, d = 0, m = 0, M = 0, nchunks = 0;
  int s = 0, nslices = 0, ngroups = 0, grid = 0;
  size_t lists_bytes = 0, partial_bytes = 0, smem = 0;
};
bool sjlt_onepass_plan(int64_t n, int64_t d, int64_t m, int s, int num_sms, const void *A, SjltOnepassPlan &p);
cudaError_t launch_sjlt_lists(const SjltOnepassPlan &p, uint64_t key, int64_t row_offset, uint16_t *lists,
                              cudaStream_t st, LaunchCounter lc);
// SA = scale * S A from the lists (partials: p.partial_bytes of scratch).
// gpart != nullptr: the gradient's partial rows g_k = sum r_i a_i ride on the
// same launch (extra warps streaming A), sjlt_onepass_grad_blocks(p) rows of d
// doubles in gpart (0: d too wide, use the separate gradient pass).
int sjlt_onepass_grad_blocks(const SjltOnepassPlan &p);
cudaError_t launch_sjlt_onepass(const SjltOnepassPlan &p, const double *A, const uint16_t *lists, double *partials,
                                double *SA, double scale, cudaStream_t st, LaunchCounter lc,
                                const double *bvec = nullptr, const double *x = nullptr, double *gpart = nullptr);
// SA[e] = scale * sum_{k < nsplit} partials[k * count + e], k ascending.
cudaError_t launch_sum_splits(const double *partials, int64_t count, int nsplit, double scale, double *SA,
                              cudaStream_t st, LaunchCounter lc);

// ---- a3 over NVLS multicast (nvls.cu) ----------------------------------------
// In-place sum of count doubles of a symmetric buffer across `world` ranks:
// mc = its multicast address, pads = device array of the world ranks' signal
// pads (unicast pointers, >= blocks * world u32 each, zero on first use).
int nvls_blocks(int64_t count, int world, int num_sms);
cudaError_t launch_nvls_allreduce(double *mc, uint32_t *const *pads, int rank, int world, int64_t count, int blocks,
                                  cudaStream_t st, LaunchCounter lc);

// ---- CSR sketch and gradient (atomics into L2) ------------------------------
// SA must be zeroed first when sketching (it receives scale * S A).  g must be zeroed when gradient.
cudaError_t launch_csr_sketch_grad(int64_t n, int64_t d, const int64_t *row_ptr, const int32_t *col,
                                   const double *val, int64_t row_offset, uint64_t key, int64_t m, int s,
                                   double scale, double *SA, const double *bvec, const double *x, double *g,
                                   cudaStream_t st, LaunchCounter lc);
cudaError_t launch_scale(double *buf, int64_t count, double scale, cudaStream_t st, LaunchCounter lc);

// ---- a5 dense gradient -------------------------------------------------------
int64_t grad_dense_blocks(int64_t n, int64_t d, int num_sms);
cudaError_t launch_grad_dense(const double *A, int64_t n, int64_t d, const double *bvec, const double *x,
                              double *gpart, int64_t nblocks, cudaStream_t st, LaunchCounter lc);
// out[c] = sum_{r < rows} part[r*d + c] (fixed order), c < d.
constexpr int64_t kReduceRowsPerCta = 64;
// scratch doubles launch_reduce_rows needs in tmp
int64_t reduce_rows_tmp(int64_t rows, int64_t d);
// out = column sums of part (rows x d), one launch, deterministic; counter: a
// device unsigned that is 0 on entry (left 0).  Hinv != nullptr: also
// x_next = x + Hinv out.  d <= 1024.
cudaError_t launch_reduce_rows(const double *part, int64_t rows, int64_t d, double *out, double *tmp,
                               unsigned *counter, cudaStream_t st, LaunchCounter lc, const double *Hinv = nullptr,
                               const double *x = nullptr, double *x_next = nullptr);

// ---- a4 Gram on DMMA ---------------------------------------------------------
struct GramPlan {
  int64_t m = 0, d = 0;
  int gt = 64;      // tile edge (64, or 128 for the large-d stream-K kernel)
  int tiles = 0;    // tiles per side (gt-wide)
  int ntri = 0;     // upper-triangular tiles
  int nsplit = 0;   // split-K
  int64_t kchunk = 0;
  int ncta = 0, kch = 0, ipc = 0;  // stream-K (ncta > 0): CTAs, k-chunks per tile, items per CTA
  size_t partial_bytes() const {
    const size_t sk = (size_t)ncta * 2 * gt * gt * 8 + (size_t)ncta * 2 * 4 + 64;
    return std::max((size_t)nsplit * ntri * 64 * 64 * 8, sk);
  }
};
// beside: the Gram shares the GPU with another kernel (the look-ahead Gram);
// for d >= 512 it then takes 128 x 128 tiles, one CTA per SM.
GramPlan gram_plan(int64_t m, int64_t d, int num_sms, int ctas_per_sm = 2, bool beside = false);
// hint = 1: SA is read with an L2 evict_first policy (stream-K plans only)
cudaError_t launch_gram(const GramPlan &p, const double *SA, double scale, double *partials, double *H,
                        cudaStream_t st, LaunchCounter lc, int hint = 0);

// ---- a6 OLS: Cholesky solve ----------------------------------------------------
// d <= 160: blocked Cholesky in one CTA (chol.cu); d > 160: ols_large.cu with
// large_mode 0 = conjugate gradients only, 1 = CG and, when CG does not finish,
// the blocked Cholesky in the same cooperative launch, 2 = the Cholesky only.
size_t chol_scratch_bytes(int64_t d);
cudaError_t launch_ols_update(const double *H, const double *g, int64_t d, const double *x, double *x_next,
                              double *scratch, int *status, int num_sms, int large_mode, cudaStream_t st,
                              LaunchCounter lc);

// a4 + a6 fused (d <= 128): H = scale^2 SA^T SA and x_next = x + H^{-1} g in one
// cluster launch; H_out (optional) receives H.
// look-ahead OLS (d <= 128): Hinv = (scale^2 SA^T SA)^{-1} in one cluster
// launch (<= max_cluster CTAs), then x_next = x + Hinv g (one CTA)
cudaError_t launch_ols_factor(const double *SA, int64_t m, int64_t d, double scale, double *Hinv, int *status,
                              int max_cluster, cudaStream_t st, LaunchCounter lc);
cudaError_t launch_ols_apply(const double *Hinv, const double *g, int64_t d, const double *x, double *x_next,
                             cudaStream_t st, LaunchCounter lc);
bool gram_ols_supported(int64_t d);
cudaError_t launch_gram_ols(const double *SA, int64_t m, int64_t d, double scale, const double *g, const double *x,
                            double *x_next, double *H_out, int *status, cudaStream_t st, LaunchCounter lc);
bool ols_large_supported(int64_t d);
size_t ols_large_scratch_bytes(int64_t d);
cudaError_t launch_ols_large(const double *H, const double *g, int64_t d, const double *x, double *x_next,
                             double *scratch, int *status, int num_sms, int mode, cudaStream_t st,
                             LaunchCounter lc);

// ---- a6 l1 ball: projected gradient -----------------------------------------
size_t pg_scratch_bytes(int64_t d);
bool pg_supported(int64_t d);
bool lasso_supported(int64_t d);
int pg_cluster_size(int64_t d);
// scratch (d doubles, may be null) keeps the power iteration's last vector;
// warm_start = it holds one from an earlier call with the same d.  prox = 1:
// the penalised form (NEXT-2), radius is lambda and the projection becomes the
// soft threshold at lambda / L (d <= 256 only: cudaErrorNotSupported beyond).
cudaError_t launch_l1ball_update(const double *H, const double *g, int64_t d, const double *x, double radius,
                                 int max_inner, int power_iters, int warm_power_iters, double tol, double safety,
                                 double *x_next,
                                 int32_t *inner_iters, double *scratch, int *status, cudaStream_t st,
                                 LaunchCounter lc, bool warm_start = false, int prox = 0,
                                 const double *L_in = nullptr, double *L_out = nullptr, int cluster_pref = 0);
// (L_in: use this step bound, no power iteration; L_out: power iteration only,
// the bound written there -- the look-ahead, api.cu; warp kernel only)

// ---- a1-a6 in one launch for small dense OLS problems (small_step.cu) --------
size_t small_step_smem(int64_t n, int64_t d, int64_t m, int s);
bool small_step_supported(int64_t n, int64_t d, int64_t m, int s);
// T iterations in one launch: x^{t+1} = x^t + H_t^{-1} g_t for H_t = (S_t A)^T S_t A,
// g_t = A^T (b - A x^t), S_t from the key of iteration iter0 + t; x^0 = x;
// x^{t+1} written to xout + t d.  SA_out / g_out / H_out (optional) receive
// the last iteration's intermediates.
cudaError_t launch_small_step(const double *A, int64_t n, int64_t d, const double *b, const double *x, uint64_t seed,
                              uint64_t iter0, int T, int64_t row_offset, int64_t m, int s, double scale, double *xout,
                              double *SA_out, double *g_out, double *H_out, int *status, cudaStream_t st,
                              LaunchCounter lc);

// ---- a7 error norms ----------------------------------------------------------
cudaError_t launch_pred_err2(int layout, int64_t n, int64_t d, const double *values, const int64_t *row_ptr,
                             const int32_t *col, const double *X, int count, const double *xref,
                             double *acc /* count+1, zeroed */, cudaStream_t st, LaunchCounter lc);

}  // namespace ihs
