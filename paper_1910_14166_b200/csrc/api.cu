// C ABI of libihs.so (include/ihs.h): context, scratch arena, argument
// validation, kernel dispatch, the IHS solve loops and the NCCL exchange.
// Every numerical step runs in the kernels of this directory.
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../../include/ihs.h"
#include "common.cuh"
#include "kernels.h"

namespace ihs {
cudaError_t launch_pred_err2_impl(int layout, int64_t n, int64_t d, const double *values, const int64_t *row_ptr,
                                  const int32_t *col, const double *X, int count, const double *xref,
                                  double *err2, double *scratch, int num_sms, cudaStream_t st, LaunchCounter lc);
}

using namespace ihs;

// ----------------------------------------------------------------------------
// NCCL, resolved at run time (the libnccl.so.2 torch already loaded).
// ----------------------------------------------------------------------------
namespace {
typedef int nccl_result;
typedef void *nccl_comm;
struct nccl_uid { char internal[128]; };
struct NcclApi {
  bool loaded = false;
  nccl_result (*GetUniqueId)(nccl_uid *) = nullptr;
  nccl_result (*CommInitRank)(nccl_comm *, int, nccl_uid, int) = nullptr;
  nccl_result (*AllReduce)(const void *, void *, size_t, int, int, nccl_comm, cudaStream_t) = nullptr;
  nccl_result (*CommDestroy)(nccl_comm) = nullptr;
};
NcclApi g_nccl;
bool load_nccl() {
  if (g_nccl.loaded) return true;
  void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return false;
  g_nccl.GetUniqueId = (nccl_result(*)(nccl_uid *))dlsym(h, "ncclGetUniqueId");
  g_nccl.CommInitRank = (nccl_result(*)(nccl_comm *, int, nccl_uid, int))dlsym(h, "ncclCommInitRank");
  g_nccl.AllReduce =
      (nccl_result(*)(const void *, void *, size_t, int, int, nccl_comm, cudaStream_t))dlsym(h, "ncclAllReduce");
  g_nccl.CommDestroy = (nccl_result(*)(nccl_comm))dlsym(h, "ncclCommDestroy");
  g_nccl.loaded = g_nccl.GetUniqueId && g_nccl.CommInitRank && g_nccl.AllReduce && g_nccl.CommDestroy;
  return g_nccl.loaded;
}
constexpr int kNcclFloat64 = 8, kNcclSum = 0;

enum Slot {
  S_PERM, S_HIST, S_TILES, S_GPART, S_GRAM, S_SJLT, S_CHOL, S_PACK, S_H, S_X, S_MISC, S_ERR,
  S_A, S_RP, S_COL, S_B, S_XH, S_X0, S_PERM2, S_HIST2, S_TILES2, S_PG, S_GRAMF, S_PGF, S_LISTS, S_ROWS, S_NSLOTS
};
}  // namespace

struct ihs_ctx_s {
  int device = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  int *d_status = nullptr;
  int64_t launches = 0;
  void *slot[S_NSLOTS] = {};
  size_t cap[S_NSLOTS] = {};
  nccl_comm comm = nullptr;
  int rank = 0, world = 1;
  ihs_status sticky = IHS_OK;
  // profiling: (group, start, stop) per timed launch; events reused after reset
  bool profiling = false;
  // Options (ihs_ctx_set_option; initial values from the IHS_* environment at
  // ihs_ctx_create).  Per context, so alternatives can be compared in one process.
  int sjlt_onepass = 1;  // dense SJLT: 1 = one read of A (sjlt_onepass.cu) with the gradient riding on it,
                         // 2 = the same with the gradient in its own pass, 0 = s sorted CountSketch passes
  int lookahead = -1;    // look-ahead schedules: -1 = by size (use_lookahead), 0 = off, 1 = whenever supported
  int ols_large = 1;     // d > 160 OLS: 0 = CG only, 1 = CG + Cholesky fallback, 2 = Cholesky only
  int fuse_max_d = 64;   // a4 + a6 in one cluster launch up to this d (<= 128)
  int pg_warm = 1;       // warm-started power iteration across l1 / LASSO updates
  int small_step = 1;    // small dense OLS solves: one launch per iteration (small_step.cu)
  int pg_cluster = 0;    // PG cluster size for d <= 256 (0: the smallest that holds H)
  int la_gram_sms = 0;   // SMs the wide (d > 256) look-ahead Gram takes (0: by the rule in gram_side_impl)
  int la_gram_tile = 0;  // its CTA tile: 0 / 64 = the 64 x 64 stream-K (two 128-thread CTAs per SM leave the
                         // pass's CTAs registers to run beside them), 128 = the 128 x 128 stream-K
  // Speculative sort of the NEXT iteration's buckets on a side stream: the
  // hash (hence the sort) depends only on (seed, iteration, row), not on x, so
  // after the gathers of iteration t the sort for t + 1 runs beside the
  // gradient reduction, Gram and inner solve of t (IHS_PREFETCH=0 disables).
  bool prefetch = true;
  cudaStream_t side = nullptr;
  cudaEvent_t ev_side = nullptr, ev_main = nullptr;
  cudaEvent_t ev_switch = nullptr;  // orders a newly bound stream after the old one
  bool side_pending = false;  // side work not yet waited on by the main stream
  struct SortTag {
    bool valid = false;
    uint64_t key = 0;
    int64_t row_offset = 0, n = 0, M = 0;
    int s = 0;
    const void *A = nullptr;
  } pre;
  int pre_set = 0;
  // Look-ahead OLS factor (ihs_ols_factor): its own high-priority stream so
  // the Gram + Cholesky + inverse of the NEXT sketch run beside this pass's
  // gather; joined into `stream` by ihs_ols_apply / synchronize / destroy.
  cudaStream_t fstream = nullptr;
  cudaEvent_t ev_fmain = nullptr;
  struct Factor {  // one in-flight factor per output buffer
    const double *Hinv = nullptr;
    cudaEvent_t done = nullptr;
    bool pending = false;
    bool L_ready = false;  // look-ahead Gram: the PG step bound of this H is in d_L[slot]
    int64_t L_d = 0;
  } fac[4];
  double *d_L = nullptr;     // [4] step bounds formed beside the pass
  int64_t pgf_warm_d = -1;   // S_PGF holds the side power iteration's vector for this d
  bool f_pending = false;  // any fac[k].pending
  int64_t pg_warm_d = -1;  // S_PG holds a power-iteration vector for this d
  struct Rec { int group; cudaEvent_t a, b; };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;
  size_t pool_used = 0;
  cudaEvent_t ev() {
    if (pool_used == pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      pool.push_back(e);
    }
    return pool[pool_used++];
  }
};

namespace {
struct DevGuard {
  int prev = -1;
  explicit DevGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DevGuard() {
    int cur;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

ihs_status from_cuda(cudaError_t e) {
  if (e == cudaSuccess) return IHS_OK;
  if (e == cudaErrorMemoryAllocation) return IHS_ERR_OUT_OF_MEMORY;
  return IHS_ERR_CUDA;
}

#define IHS_TRY(expr)                         \
  do {                                        \
    ihs_status _s = (expr);                   \
    if (_s != IHS_OK) return _s;              \
  } while (0)
#define IHS_CUDA(expr) IHS_TRY(from_cuda(expr))

void join_side(ihs_ctx c);
void join_factor(ihs_ctx c);

// The collective schedules run whenever the ctx holds a communicator -- also a
// one-rank one (ihs_ctx_set_comm(c, 0, 1, uid)), whose all-reduces are NCCL
// calls over one rank: the multi-rank plumbing exercised on one GPU.
inline bool distributed(const ihs_ctx_s *c) { return c->world > 1 || c->comm != nullptr; }

template <typename T>
ihs_status scratch(ihs_ctx c, Slot s, size_t bytes, T **out) {
  bytes = std::max<size_t>(bytes, 256);
  if (c->cap[s] < bytes) {
    join_side(c);  // the side stream may still use this slot
    join_factor(c);  // so may the factor stream (S_PACK)
    if (c->slot[s]) {
      cudaError_t e = cudaFreeAsync(c->slot[s], c->stream);
      if (e != cudaSuccess) return from_cuda(e);
      c->slot[s] = nullptr;
      c->cap[s] = 0;
    }
    size_t want = bytes + bytes / 8;
    void *p = nullptr;
    cudaError_t e = cudaMallocAsync(&p, want, c->stream);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return IHS_ERR_OUT_OF_MEMORY;
    }
    c->slot[s] = p;
    c->cap[s] = want;
  }
  *out = reinterpret_cast<T *>(c->slot[s]);
  return IHS_OK;
}

LaunchCounter lc_of(ihs_ctx c) { return LaunchCounter{&c->launches}; }

// RAII: events around one kernel-group launch when profiling is on.
struct Prof {
  ihs_ctx c;
  int group;
  cudaStream_t st;
  cudaEvent_t b = nullptr;
  Prof(ihs_ctx c_, int g, cudaStream_t s_ = nullptr) : c(c_), group(g), st(s_ ? s_ : c_->stream) {
    if (c->profiling) {
      cudaEvent_t a = c->ev();
      b = c->ev();
      cudaEventRecord(a, st);
      c->recs.push_back({group, a, b});
    }
  }
  ~Prof() {
    if (b) cudaEventRecord(b, st);
  }
};

// The main stream waits for any side-stream work issued earlier (before it
// touches, frees or regrows the buffers the side stream writes).
void join_side(ihs_ctx c) {
  if (c->side_pending) {
    cudaStreamWaitEvent(c->stream, c->ev_side, 0);
    c->side_pending = false;
  }
}

void join_factor(ihs_ctx c) {
  if (c->f_pending) {
    for (auto &f : c->fac)
      if (f.pending) {
        cudaStreamWaitEvent(c->stream, f.done, 0);
        f.pending = false;
      }
    c->f_pending = false;
  }
}

ihs_status check_spec(const ihs_sketch_spec *spec) {
  if (!spec) return IHS_ERR_INVALID_ARGUMENT;
  if (spec->m < 1 || spec->s < 1) return IHS_ERR_INVALID_ARGUMENT;
  if (spec->family == IHS_COUNTSKETCH) {
    if (spec->s != 1) return IHS_ERR_INVALID_ARGUMENT;
  } else if (spec->family == IHS_SJLT) {
    if (spec->s > spec->m) return IHS_ERR_INVALID_ARGUMENT;
    if (spec->m % spec->s != 0) return IHS_ERR_DIMENSION_MISMATCH;
  } else {
    return IHS_ERR_INVALID_ARGUMENT;
  }
  if (spec->m / spec->s > 0xffffffffLL || spec->m > (int64_t(1) << 31)) return IHS_ERR_UNSUPPORTED;
  return IHS_OK;
}

ihs_status check_matrix(const ihs_matrix *A) {
  if (!A || A->reserved != 0) return IHS_ERR_INVALID_ARGUMENT;
  if (A->n_rows < 0 || A->n_cols < 1 || A->row_offset < 0) return IHS_ERR_INVALID_ARGUMENT;
  if (A->n_rows >= (int64_t(1) << 31)) return IHS_ERR_UNSUPPORTED;
  if (A->layout == IHS_DENSE_ROW_MAJOR) {
    if (A->n_rows > 0 && !A->values) return IHS_ERR_INVALID_ARGUMENT;
    if (A->n_cols > (int64_t(1) << 30)) return IHS_ERR_UNSUPPORTED;
  } else if (A->layout == IHS_CSR) {
    if (!A->row_ptr || A->nnz < 0) return IHS_ERR_INVALID_ARGUMENT;
    if (A->nnz > 0 && (!A->values || !A->col_idx)) return IHS_ERR_INVALID_ARGUMENT;
  } else {
    return IHS_ERR_INVALID_ARGUMENT;
  }
  return IHS_OK;
}

double spec_scale(const ihs_sketch_spec *spec) { return spec->s > 1 ? 1.0 / std::sqrt((double)spec->s) : 1.0; }

// ---- a2 (and a5 when g != null), local partials ------------------------------
unsigned *reduce_counter(ihs_ctx c) { return reinterpret_cast<unsigned *>(c->d_status + 1); }

// One look-ahead OLS step riding on a pass (no all-reduce between the pass and
// the update, i.e. one rank): after the gathers, the factor of this pass's SA
// (S^{t+1} A) is enqueued into Hinv_next (if set); the gradient reduction then
// also applies x_next = x + Hinv g in its last CTA (one launch).
struct LookStep {
  const double *Hinv;
  const double *x;
  double *x_next;
  double *Hinv_next;
};
ihs_status ols_factor_impl(ihs_ctx c, const double *SA, int64_t m, int64_t d, double scale, double *Hinv);
ihs_status wait_factor(ihs_ctx c, const double *Hinv);
ihs_status ols_apply_impl(ihs_ctx c, const double *Hinv, const double *g, int64_t d, const double *x, double *xn);

// The side stream (sort prefetch, SJLT lists), created on first use at low
// priority: its CTAs take the slots the HBM-bound passes leave.
ihs_status ensure_side(ihs_ctx c) {
  if (!c->side) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    IHS_CUDA(cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, lo));
    IHS_CUDA(cudaEventCreateWithFlags(&c->ev_side, cudaEventDisableTiming));
    IHS_CUDA(cudaEventCreateWithFlags(&c->ev_main, cudaEventDisableTiming));
  }
  return IHS_OK;
}

ihs_status sketch_grad_impl(ihs_ctx c, const ihs_matrix *A, const ihs_sketch_spec *spec, uint64_t iter,
                            const double *b, const double *x, double *SA, double *g, const LookStep *ls = nullptr) {
  const uint64_t key = iter_key(spec->seed, iter);
  const int64_t n = A->n_rows, d = A->n_cols, m = spec->m;
  const int s = spec->s;
  cudaStream_t st = c->stream;
  if (A->layout == IHS_CSR) {
    if (SA) IHS_CUDA(cudaMemsetAsync(SA, 0, (size_t)m * d * 8, st));
    if (g) IHS_CUDA(cudaMemsetAsync(g, 0, (size_t)d * 8, st));
    {
      Prof pr(c, IHS_K_CSR);
      IHS_CUDA(launch_csr_sketch_grad(n, d, A->row_ptr, A->col_idx, A->values, A->row_offset, key, m, s,
                                      spec_scale(spec), SA, b, x, g, st, lc_of(c)));
    }
    return IHS_OK;
  }
  // dense.  CountSketch (s = 1): a stable counting sort of the rows by bucket
  // and one bucket-ordered gather, with the gradient riding on the same read
  // of A.  SJLT (s > 1): the same per block j (s stacked
  // CountSketches; s reads of A, bit-identical to the oracle) when the
  // "sjlt_onepass" option is 0; by default one read of A (below).
  const int64_t M = m / s;
  SjltOnepassPlan op;
  if (SA && s > 1 && c->sjlt_onepass && n > 0 && sjlt_onepass_plan(n, d, m, s, c->num_sms, A->values, op)) {
    // One read of A for S A (sjlt_onepass.cu): the per-chunk bucket lists
    // (a1), then the column-slice sketch pass with the gradient (a5) riding on
    // it in extra warps (C5: 21.1 + 4.3 ms in two passes -> 22.9 ms).  (A
    // separate co-resident gradient kernel could not share the SMs: the
    // sketch's 17 warps leave an SM sub-partition 1 K registers, and an SM
    // that started the small kernel first is carved out for L1.)
    join_side(c);
    join_factor(c);
    uint16_t *lists;
    double *part;
    IHS_TRY(scratch(c, S_LISTS, op.lists_bytes, &lists));
    IHS_TRY(scratch(c, S_SJLT, op.partial_bytes, &part));
    IHS_TRY(ensure_side(c));
    c->pre.valid = false;
    IHS_CUDA(cudaEventRecord(c->ev_main, st));
    IHS_CUDA(cudaStreamWaitEvent(c->side, c->ev_main, 0));
    {
      Prof pr(c, IHS_K_SORT, c->side);
      IHS_CUDA(launch_sjlt_lists(op, key, A->row_offset, lists, c->side, lc_of(c)));
    }
    IHS_CUDA(cudaEventRecord(c->ev_side, c->side));
    c->side_pending = true;
    // The gradient (a5) rides on the sketch pass by default: extra warps of
    // its CTAs stream A for g (sjlt_onepass.cu), hidden under the sketch's
    // shared-memory-bound work.  Option sjlt_onepass = 2, or d > 128: the
    // gradient in its own pass beside the lists instead.
    const int nfused = (g && c->sjlt_onepass == 1) ? sjlt_onepass_grad_blocks(op) : 0;
    const int64_t nbg = nfused ? nfused : grad_dense_blocks(n, d, c->num_sms);
    double *gpart = nullptr;
    if (g) {
      if (d > 1024) return IHS_ERR_UNSUPPORTED;
      IHS_TRY(scratch(c, S_GPART, ((size_t)nbg * d + reduce_rows_tmp(nbg, d)) * 8, &gpart));
    }
    if (g && !nfused) {
      Prof pr(c, IHS_K_GRAD);
      IHS_CUDA(launch_grad_dense(A->values, n, d, b, x, gpart, nbg, st, lc_of(c)));
    }
    join_side(c);
    {
      Prof pr(c, IHS_K_SJLT);
      IHS_CUDA(launch_sjlt_onepass(op, A->values, lists, part, SA, spec_scale(spec), st, lc_of(c), nfused ? b : nullptr,
                                   nfused ? x : nullptr, nfused ? gpart : nullptr));
    }
    if (g) {
      if (ls && ls->Hinv_next) IHS_TRY(ols_factor_impl(c, SA, m, d, 1.0, ls->Hinv_next));
      if (ls) IHS_TRY(wait_factor(c, ls->Hinv));
      Prof pr(c, ls ? IHS_K_APPLY : IHS_K_REDUCE);
      IHS_CUDA(launch_reduce_rows(gpart, nbg, d, g, gpart + nbg * d, reduce_counter(c), st, lc_of(c),
                                  ls ? ls->Hinv : nullptr, ls ? ls->x : nullptr, ls ? ls->x_next : nullptr));
    }
    return IHS_OK;
  }
  const bool use_sort = cs_sort_supported(M);
  const bool fuse = SA && use_sort && g && d <= 256;
  if (SA) {
    if (use_sort) {
      CsSortPlan p = cs_sort_plan(n, M);
      // SJLT blocks are gathered nb at a time (one launch, grid.y = block) so
      // that a launch has about two waves of bucket CTAs (7 per SM resident)
      // even when M = m / s is small: the gradient-carrying block's slower CTAs
      // then share a launch with three others (C5: 35.4 -> 34.4 ms/step against
      // one wave).  The sort buffers hold all s blocks; two sets, so
      // the next iteration's sort can be prefetched into the other set.
      const bool tma = cs_gather_tma_supported(d, A->values);
      const int nb = !tma ? 1
                          : (int)std::max<int64_t>(1, std::min<int64_t>(s, (14 * (int64_t)c->num_sms) / std::max<int64_t>(M, 1)));
      const int64_t hs = (int64_t)(p.hist_bytes() / 4 + 63) / 64 * 64, ts = (int64_t)(p.tiles_bytes() / 4 + 63) / 64 * 64;
      const int64_t ps = (p.n + 63) / 64 * 64;
      const bool hit = c->pre.valid && c->pre.key == key && c->pre.row_offset == A->row_offset && c->pre.n == n &&
                       c->pre.M == M && c->pre.s == s && c->pre.A == (const void *)A->values;
      join_side(c);  // also orders any scratch (re)allocation below after side-stream use
      const int set = hit ? c->pre_set : (c->pre.valid ? 1 - c->pre_set : 0);
      c->pre.valid = false;
      int32_t *hist, *tiles;
      uint32_t *perm;
      auto get_set = [&](int k, int32_t **h, int32_t **t, uint32_t **pm) -> ihs_status {
        IHS_TRY(scratch(c, k ? S_HIST2 : S_HIST, (size_t)hs * 4 * s, h));
        IHS_TRY(scratch(c, k ? S_TILES2 : S_TILES, (size_t)ts * 4 * s, t));
        return scratch(c, k ? S_PERM2 : S_PERM, (size_t)std::max<int64_t>(ps, 1) * 4 * s, pm);
      };
      IHS_TRY(get_set(set, &hist, &tiles, &perm));
      auto sort_all = [&](uint64_t k, int32_t *h, int32_t *t, uint32_t *pm, cudaStream_t sst) -> ihs_status {
        Prof pr(c, IHS_K_SORT, sst);
        for (int j = 0; j < s; ++j)
          IHS_CUDA(launch_cs_sort(p, k, A->row_offset, (uint32_t)j, (uint32_t)s, h + j * hs, t + j * ts, pm + j * ps,
                                  sst, lc_of(c)));
        return IHS_OK;
      };
      if (!hit) IHS_TRY(sort_all(key, hist, tiles, perm, st));
      // few buckets with long row lists (small m): split every bucket's rows
      // into nseg segments (grid.z) so a launch still fills the GPU; the
      // segment partials are summed in order afterwards (SA then agrees with
      // the oracle to rounding instead of bit for bit, R3)
      int nseg = 1;
      if (tma && M * nb < 4 * (int64_t)c->num_sms && n / std::max<int64_t>(M, 1) >= 1024)
        nseg = (int)std::max<int64_t>(1, std::min<int64_t>((7 * (int64_t)c->num_sms + M * nb - 1) / (M * nb),
                                                           n / (M * 512)));
      double *gpart = nullptr;
      if (fuse)
        IHS_TRY(scratch(c, S_GPART, ((size_t)M * d * nseg + reduce_rows_tmp(M * nseg, d)) * 8, &gpart));
      double *sapart = nullptr;
      if (nseg > 1) IHS_TRY(scratch(c, S_SJLT, (size_t)nseg * nb * M * d * 8, &sapart));
      const double scale = spec_scale(spec);
      // Speculative prefetch of iteration iter + 1 into the other set, on the
      // side stream, concurrent with this iteration's gathers: the sort kernels
      // (hash + smem histogram + scatter, compute/L2-bound) co-reside with the
      // HBM-bound gather CTAs, so the next sort is hidden behind this
      // iteration's read of A.  The other set was last read by the gathers of
      // iter - 1, which precede ev_main on the main stream.
      // The side-stream sort is enqueued after the first gather launch (still
      // eligible from ev_main, recorded before it), so the gather's CTAs are
      // placed first and the sort takes leftover slots: C2 0.794 -> 0.789,
      // C4 0.859 -> 0.848, C5 36.9 -> 36.1 ms/step against enqueueing it first.
      // The ctx records the prefetch (pre, side_pending) only once its sort is
      // enqueued, so a failed launch before it leaves no stale tag behind.
      bool pf_pending = false;
      uint64_t pf_key = 0;
      int32_t *pf_h = nullptr, *pf_t = nullptr;
      uint32_t *pf_p = nullptr;
      ihs_ctx_s::SortTag pf_tag;
      int pf_set = 0;
      auto issue_prefetch = [&]() -> ihs_status {
        pf_pending = false;
        IHS_TRY(sort_all(pf_key, pf_h, pf_t, pf_p, c->side));
        IHS_CUDA(cudaEventRecord(c->ev_side, c->side));
        c->side_pending = true;
        c->pre = pf_tag;
        c->pre_set = pf_set;
        return IHS_OK;
      };
      if (c->prefetch && n > 0) {
        IHS_TRY(ensure_side(c));
        const int nset = 1 - set;
        int32_t *h2, *t2;
        uint32_t *p2;
        IHS_TRY(get_set(nset, &h2, &t2, &p2));  // allocated on the main stream, before ev_main
        IHS_CUDA(cudaEventRecord(c->ev_main, st));
        IHS_CUDA(cudaStreamWaitEvent(c->side, c->ev_main, 0));
        const uint64_t key_next = iter_key(spec->seed, iter + 1);
        pf_key = key_next;
        pf_h = h2;
        pf_t = t2;
        pf_p = p2;
        pf_pending = true;
        pf_tag.valid = true;
        pf_tag.key = key_next;
        pf_tag.row_offset = A->row_offset;
        pf_tag.n = n;
        pf_tag.M = M;
        pf_tag.s = s;
        pf_tag.A = A->values;
        pf_set = nset;
      }
      for (int j0 = 0; j0 < s; j0 += nb) {
        const int cnt = std::min(nb, s - j0);
        int32_t *hist_j = hist + j0 * hs, *tiles_j = tiles + j0 * ts;
        uint32_t *perm_j = perm + j0 * ps;
        double *SAj = SA + (int64_t)j0 * M * d;
        double *gp = (j0 == 0) ? gpart : nullptr;
        Prof pr(c, IHS_K_SKETCH);
        if (tma) {
          GatherBatchStrides bst;
          bst.hist = hs;
          bst.tiles = ts;
          bst.perm = ps;
          bst.sa = M * d;
          bst.nseg = nseg;
          bst.seg_sa = (int64_t)cnt * M * d;
          IHS_CUDA(launch_cs_gather_tma(A->values, n, d, M, hist_j, tiles_j, p.nchunks, perm_j, b, x,
                                        nseg > 1 ? sapart : SAj, gp, nseg > 1 ? 1.0 : scale, st, lc_of(c), cnt, bst));
          if (nseg > 1)
            IHS_CUDA(launch_sum_splits(sapart, (int64_t)cnt * M * d, nseg, scale, SAj, st, lc_of(c)));
        } else {  // odd d, d > 256 or an unaligned A: the register-staged gather
          IHS_CUDA(launch_cs_gather(A->values, n, d, M, hist_j, tiles_j, p.nchunks, perm_j, b, x, SAj, gp, scale, st,
                                    lc_of(c)));
        }
        if (pf_pending) IHS_TRY(issue_prefetch());
      }
      if (fuse) {
        if (ls && ls->Hinv_next) IHS_TRY(ols_factor_impl(c, SA, m, d, 1.0, ls->Hinv_next));
        if (ls) IHS_TRY(wait_factor(c, ls->Hinv));
        Prof pr(c, ls ? IHS_K_APPLY : IHS_K_REDUCE);
        IHS_CUDA(launch_reduce_rows(gpart, M * nseg, d, g, gpart + M * nseg * d, reduce_counter(c), st, lc_of(c),
                                    ls ? ls->Hinv : nullptr, ls ? ls->x : nullptr, ls ? ls->x_next : nullptr));
      }
    } else {  // more buckets than the counting sort handles: shared-memory tiles (sjlt_dense.cu)
      SjltPlan p;
      if (!sjlt_plan(n, d, m, s, c->num_sms, p)) return IHS_ERR_UNSUPPORTED;
      double *part;
      IHS_TRY(scratch(c, S_SJLT, p.partial_bytes(), &part));
      Prof pr(c, IHS_K_SJLT);
      IHS_CUDA(launch_sjlt_dense(p, A->values, key, A->row_offset, part, SA, spec_scale(spec), st, lc_of(c)));
    }
  }
  if (g && !fuse) {
    if (d > 1024) return IHS_ERR_UNSUPPORTED;
    const int64_t nb = grad_dense_blocks(n, d, c->num_sms);
    double *gpart;
    IHS_TRY(scratch(c, S_GPART, ((size_t)nb * d + reduce_rows_tmp(nb, d)) * 8, &gpart));
    if (n == 0) {
      IHS_CUDA(cudaMemsetAsync(g, 0, (size_t)d * 8, st));
      if (ls && ls->Hinv_next && SA) IHS_TRY(ols_factor_impl(c, SA, m, d, 1.0, ls->Hinv_next));
      if (ls) IHS_TRY(ols_apply_impl(c, ls->Hinv, g, d, ls->x, ls->x_next));
    } else {
      {
        Prof pr(c, IHS_K_GRAD);
        IHS_CUDA(launch_grad_dense(A->values, n, d, b, x, gpart, nb, st, lc_of(c)));
      }
      if (ls && ls->Hinv_next && SA) IHS_TRY(ols_factor_impl(c, SA, m, d, 1.0, ls->Hinv_next));
      if (ls) IHS_TRY(wait_factor(c, ls->Hinv));
      Prof pr(c, ls ? IHS_K_APPLY : IHS_K_REDUCE);
      IHS_CUDA(launch_reduce_rows(gpart, nb, d, g, gpart + nb * d, reduce_counter(c), st, lc_of(c),
                                  ls ? ls->Hinv : nullptr, ls ? ls->x : nullptr, ls ? ls->x_next : nullptr));
    }
  }
  return IHS_OK;
}

ihs_status gram_impl(ihs_ctx c, const double *SA, int64_t m, int64_t d, double scale, double *H) {
  GramPlan p = gram_plan(m, d, c->num_sms);
  double *part;
  IHS_TRY(scratch(c, S_GRAM, p.partial_bytes(), &part));
  Prof pr(c, IHS_K_GRAM);
  IHS_CUDA(launch_gram(p, SA, scale, part, H, c->stream, lc_of(c)));
  return IHS_OK;
}

ihs_status ols_impl(ihs_ctx c, const double *H, const double *g, int64_t d, const double *x, double *xn) {
  IHS_TRY(wait_factor(c, H));
  double *sc;
  IHS_TRY(scratch(c, S_CHOL, chol_scratch_bytes(d), &sc));
  Prof pr(c, IHS_K_CHOL);
  IHS_CUDA(launch_ols_update(H, g, d, x, xn, sc, c->d_status, c->num_sms, c->ols_large, c->stream, lc_of(c)));
  return IHS_OK;
}

// a4 + a6 (OLS) in one cluster launch.  Measured on B200: a win while launch
// latency dominates (C1, d = 10: 31 -> 21 us) but not at d = 96..128 (C2: 69 ->
// 73 us, C5: 67 -> 97 us: the DSMEM reduction runs at 14-30 GB/s per SM), so
// the default fuses only d <= 64; IHS_FUSE=1 forces it for d <= 128, 0 never.
ihs_status gram_ols_impl(ihs_ctx c, const double *SA, int64_t m, int64_t d, double scale, const double *g,
                         const double *x, double *xn, double *H) {
  if (d <= c->fuse_max_d && gram_ols_supported(d) && m >= 1) {
    Prof pr(c, IHS_K_CHOL);
    const cudaError_t e = launch_gram_ols(SA, m, d, scale, g, x, xn, H, c->d_status, c->stream, lc_of(c));
    if (e == cudaSuccess) return IHS_OK;
    cudaGetLastError();  // cluster launch refused: the two-call path below
  }
  IHS_TRY(gram_impl(c, SA, m, d, scale, H));
  return ols_impl(c, H, g, d, x, xn);
}

// Look-ahead OLS, part 1: Hinv = (scale^2 SA^T SA)^{-1} on the factor stream,
// ordered after everything already enqueued on the ctx stream.  Completion is
// tracked per output buffer, so ihs_ols_apply on the previous buffer does not
// wait for this factor (the look-ahead loop enqueues the factor of S^{t+1}
// before the apply of H_t^{-1}, so that its cluster is placed before the next
// pass's gather fills the SMs).
// The factor stream, ordered after everything already on the ctx stream; the
// returned record gets the completion event of the work enqueued next.
ihs_status factor_begin(ihs_ctx c, const double *out, ihs_ctx_s::Factor **rec) {
  if (!c->fstream) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    IHS_CUDA(cudaStreamCreateWithPriority(&c->fstream, cudaStreamNonBlocking, hi));
    IHS_CUDA(cudaEventCreateWithFlags(&c->ev_fmain, cudaEventDisableTiming));
    for (auto &f : c->fac) IHS_CUDA(cudaEventCreateWithFlags(&f.done, cudaEventDisableTiming));
  }
  ihs_ctx_s::Factor *slot = nullptr;
  for (auto &f : c->fac)
    if (f.pending && f.Hinv == out) slot = &f;  // a rewrite of the same buffer: fstream order suffices
  if (!slot)
    for (auto &f : c->fac)
      if (!f.pending) {
        slot = &f;
        break;
      }
  if (!slot) {
    join_factor(c);
    slot = &c->fac[0];
  }
  IHS_CUDA(cudaEventRecord(c->ev_fmain, c->stream));
  IHS_CUDA(cudaStreamWaitEvent(c->fstream, c->ev_fmain, 0));
  slot->L_ready = false;  // (set again by a look-ahead Gram that also forms the step bound)
  *rec = slot;
  return IHS_OK;
}

ihs_status factor_end(ihs_ctx c, const double *out, ihs_ctx_s::Factor *slot) {
  IHS_CUDA(cudaEventRecord(slot->done, c->fstream));
  slot->Hinv = out;
  slot->pending = true;
  c->f_pending = true;
  return IHS_OK;
}

// Look-ahead Gram for the l1 / LASSO updates: H = scale^2 SA^T SA on the factor
// stream with a Gram plan for a few SMs (it runs beside the previous update's
// PG cluster; the update that reads H joins it).
ihs_inner_cfg default_inner();

ihs_status gram_side_impl(ihs_ctx c, const double *SA, int64_t m, int64_t d, double scale, double *H) {
  if (m < 1 || d < 1) return IHS_ERR_INVALID_ARGUMENT;
  // d <= 256 (the l1 / LASSO updates): a 16-SM plan, beside the update's
  // cluster; larger d (OLS with the CG update, e.g. C3): a full plan reading
  // SA evict_first, beside the CG solve and the next pass's L2 reductions
  const bool wide = d > 256;
  // A 128-tile Gram CTA holds a whole SM's register file (512 threads x 128 registers), so
  // no CTA of the pass runs on that SM while it is there: beside the pass the two merely
  // queue (C3, K consecutive steps: 0.71 ms/step).  The 64-tile stream-K (2 x 128 threads x
  // 152 registers per SM) leaves the pass room: 0.63; either tile on a share of the SMs
  // ("la_gram_sms") measured 0.62-0.64 (profiles/r02/c3_lookahead_gram_sweep.json)
  const int wide_sms = c->la_gram_sms > 0 ? std::min(c->la_gram_sms, c->num_sms) : c->num_sms;
  GramPlan p = gram_plan(m, d, wide ? std::max(64, wide_sms) : std::min(16, c->num_sms), 2,
                         wide && c->la_gram_tile == 128);
  double *part;
  IHS_TRY(scratch(c, S_GRAMF, p.partial_bytes(), &part));  // (before factor_begin: a regrowth joins)
  const bool power = pg_supported(d);
  double *ev = nullptr;
  if (power) {  // allocated on the ctx stream before the factor stream's dependency is recorded
    if (!c->d_L) IHS_CUDA(cudaMalloc(&c->d_L, 4 * sizeof(double)));
    if (c->cap[S_PGF] < std::max<size_t>(pg_scratch_bytes(d), 256)) c->pgf_warm_d = -1;
    IHS_TRY(scratch(c, S_PGF, pg_scratch_bytes(d), &ev));
  }
  ihs_ctx_s::Factor *slot;
  IHS_TRY(factor_begin(c, H, &slot));
  {
    Prof pr(c, IHS_K_FACTOR, c->fstream);
    IHS_CUDA(launch_gram(p, SA, scale, part, H, c->fstream, lc_of(c), wide ? 1 : 0));
  }
  // ... and the PG step bound L = 1.05 lambda_max(H) (R10's power iteration,
  // warm-started along the chain of look-ahead Grams exactly as the update
  // would have), so the update of this H skips its power steps
  slot->L_ready = false;
  if (power) {
    const ihs_inner_cfg k = default_inner();
    Prof pr(c, IHS_K_FACTOR, c->fstream);
    const cudaError_t e = launch_l1ball_update(H, nullptr, d, nullptr, 0.0, 0, k.power_iters, k.warm_power_iters,
                                               k.inner_tol, k.lip_safety, nullptr, nullptr, ev, c->d_status,
                                               c->fstream, lc_of(c), c->pgf_warm_d == d, 0, nullptr,
                                               c->d_L + (slot - c->fac), c->pg_cluster);
    if (e == cudaSuccess) {
      c->pgf_warm_d = d;
      slot->L_ready = true;
      slot->L_d = d;
    } else {
      cudaGetLastError();
    }
  }
  return factor_end(c, H, slot);
}

ihs_status ols_factor_impl(ihs_ctx c, const double *SA, int64_t m, int64_t d, double scale, double *Hinv) {
  if (!gram_ols_supported(d) || m < 1) return IHS_ERR_UNSUPPORTED;
  ihs_ctx_s::Factor *slot;
  IHS_TRY(factor_begin(c, Hinv, &slot));
  {
    Prof pr(c, IHS_K_FACTOR, c->fstream);
    IHS_CUDA(launch_ols_factor(SA, m, d, scale, Hinv, c->d_status, 8, c->fstream, lc_of(c)));
  }
  return factor_end(c, Hinv, slot);
}

// Look-ahead OLS, part 2: x_next = x + Hinv g on the ctx stream, after the
// pending factor that writes Hinv (if any).
ihs_status wait_factor(ihs_ctx c, const double *Hinv) {
  for (auto &f : c->fac)
    if (f.pending && f.Hinv == Hinv) {
      IHS_CUDA(cudaStreamWaitEvent(c->stream, f.done, 0));
      f.pending = false;
    }
  return IHS_OK;
}

ihs_status ols_apply_impl(ihs_ctx c, const double *Hinv, const double *g, int64_t d, const double *x, double *xn) {
  IHS_TRY(wait_factor(c, Hinv));
  Prof pr(c, IHS_K_APPLY);
  IHS_CUDA(launch_ols_apply(Hinv, g, d, x, xn, c->stream, lc_of(c)));
  return IHS_OK;
}

ihs_inner_cfg default_inner() {
  ihs_inner_cfg k;
  k.max_inner = 20000;
  k.power_iters = 50;
  k.warm_power_iters = 12;
  k.reserved = 0;
  k.inner_tol = 1e-14;
  k.lip_safety = 1.05;
  return k;
}

// prox = 0: l1 ball of radius `radius`; prox = 1: penalty lambda = `radius` (NEXT-2)
ihs_status l1_impl(ihs_ctx c, const double *H, const double *g, int64_t d, const double *x, double radius,
                   const ihs_inner_cfg *cfg, double *xn, int32_t *inner, int prox = 0) {
  ihs_inner_cfg k = cfg ? *cfg : default_inner();
  if (k.max_inner < 1 || k.power_iters < 1 || k.warm_power_iters < 1 || !(k.inner_tol >= 0.0) ||
      !(k.lip_safety > 0.0))
    return IHS_ERR_INVALID_ARGUMENT;
  if (!pg_supported(d) || (prox && !lasso_supported(d))) return IHS_ERR_UNSUPPORTED;
  IHS_TRY(wait_factor(c, H));  // a look-ahead Gram that writes H
  const double *L_in = nullptr;  // ... and its step bound, formed beside the pass
  for (auto &f : c->fac)
    if (f.L_ready && f.Hinv == H) {
      const ihs_inner_cfg k0 = default_inner();
      if (f.L_d == d && k.power_iters == k0.power_iters && k.warm_power_iters == k0.warm_power_iters &&
          k.lip_safety == k0.lip_safety)
        L_in = c->d_L + (&f - c->fac);
      f.L_ready = false;
    }
  // warm-started power iteration across calls with the same d (option pg_warm)
  const bool warm_env = c->pg_warm != 0;
  double *ev = nullptr;
  if (warm_env && c->cap[S_PG] < std::max<size_t>(pg_scratch_bytes(d), 256)) c->pg_warm_d = -1;  // (re)allocation loses it
  if (warm_env) IHS_TRY(scratch(c, S_PG, pg_scratch_bytes(d), &ev));
  const bool warm = warm_env && c->pg_warm_d == d;
  Prof pr(c, IHS_K_PG);
  IHS_CUDA(launch_l1ball_update(H, g, d, x, radius, k.max_inner, k.power_iters, k.warm_power_iters, k.inner_tol,
                                k.lip_safety, xn, inner, ev, c->d_status, c->stream, lc_of(c), warm, prox, L_in,
                                nullptr, c->pg_cluster));
  if (warm_env && !L_in) c->pg_warm_d = d;
  return IHS_OK;
}

bool is_host_ptr(const void *p) {
  if (!p) return false;
  cudaPointerAttributes a;
  cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered || a.type == cudaMemoryTypeHost;
}

ihs_status sync_status(ihs_ctx c) {
  join_factor(c);
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return from_cuda(e);
  int st = 0;
  e = cudaMemcpy(&st, c->d_status, sizeof(int), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return from_cuda(e);
  if (st != 0) {
    int zero = 0;
    cudaMemcpy(c->d_status, &zero, sizeof(int), cudaMemcpyHostToDevice);
  }
  return (ihs_status)st;
}

// Look-ahead OLS loop (ihs_ols_factor / ihs_ols_apply):
// a prologue pass forms S^{iter0} A and its H^{-1}; pass t then reads A once
// for [S^{t+1} A | g^t] (one all-reduce), applies x^{t+1} = x^t + H_t^{-1} g^t,
// and factorises H_{t+1} on the factor stream beside pass t + 1.  The last
// pass forms g only.  T + 1 passes over A for T iterations, none of the d x d
// work on the critical path but the apply.
ihs_status ols_lookahead_loop(ihs_ctx c, const ihs_matrix *A, const ihs_sketch_spec *spec, const double *b,
                              uint64_t iter0, int32_t T, double *xh) {
  const int64_t d = A->n_cols, m = spec->m, pk = m * d + d;
  double *packs, *Hinv;
  IHS_TRY(scratch(c, S_PACK, (size_t)2 * pk * 8, &packs));
  IHS_TRY(scratch(c, S_H, (size_t)2 * d * d * 8, &Hinv));
  auto allreduce = [&](double *buf, int64_t cnt) -> ihs_status {
    if (distributed(c)) {
      if (!c->comm || !load_nccl()) return IHS_ERR_COMM;
      if (g_nccl.AllReduce(buf, buf, (size_t)cnt, kNcclFloat64, kNcclSum, c->comm, c->stream) != 0)
        return IHS_ERR_COMM;
    }
    return IHS_OK;
  };
  IHS_TRY(sketch_grad_impl(c, A, spec, iter0, nullptr, nullptr, packs, nullptr));
  IHS_TRY(allreduce(packs, m * d));
  IHS_TRY(ols_factor_impl(c, packs, m, d, 1.0, Hinv));
  for (int32_t t = 0; t < T; ++t) {
    const int cur = t & 1, nxt = cur ^ 1;
    const bool more = t + 1 < T;
    double *SAn = packs + nxt * pk, *gn = SAn + m * d;
    const double *x = xh + (int64_t)t * d;
    double *xn = xh + (int64_t)(t + 1) * d;
    if (!distributed(c)) {  // factor, gradient reduction and update inside the pass
      const LookStep ls{Hinv + cur * d * d, x, xn, more ? Hinv + nxt * d * d : nullptr};
      IHS_TRY(sketch_grad_impl(c, A, spec, iter0 + (uint64_t)t + 1, b, x, more ? SAn : nullptr, gn, &ls));
      continue;
    }
    IHS_TRY(sketch_grad_impl(c, A, spec, iter0 + (uint64_t)t + 1, b, x, more ? SAn : nullptr, gn));
    IHS_TRY(more ? allreduce(SAn, pk) : allreduce(gn, d));
    if (more) IHS_TRY(ols_factor_impl(c, SAn, m, d, 1.0, Hinv + nxt * d * d));
    IHS_TRY(ols_apply_impl(c, Hinv + cur * d * d, gn, d, x, xn));
  }
  return IHS_OK;
}

// Look-ahead for the l1 ball / LASSO (prox 0 / 1), and the Gram-only form for
// OLS with d > 256 (prox -1): the Gram of S^{t+1} A (formed by pass t with g^t)
// runs on the factor stream beside the update of iteration t and the next
// pass; the update of t + 1 then finds H_{t+1} ready.  T + 1 passes.
ihs_status pg_lookahead_loop(ihs_ctx c, const ihs_matrix *A, const ihs_sketch_spec *spec, const double *b,
                             uint64_t iter0, int32_t T, double *xh, double radius, const ihs_inner_cfg *cfg,
                             int32_t *inner_dev, int prox) {
  const int64_t d = A->n_cols, m = spec->m, pk = m * d + d;
  double *packs, *H;
  IHS_TRY(scratch(c, S_PACK, (size_t)2 * pk * 8, &packs));
  IHS_TRY(scratch(c, S_H, (size_t)2 * d * d * 8, &H));
  auto allreduce = [&](double *buf, int64_t cnt) -> ihs_status {
    if (distributed(c)) {
      if (!c->comm || !load_nccl()) return IHS_ERR_COMM;
      if (g_nccl.AllReduce(buf, buf, (size_t)cnt, kNcclFloat64, kNcclSum, c->comm, c->stream) != 0)
        return IHS_ERR_COMM;
    }
    return IHS_OK;
  };
  IHS_TRY(sketch_grad_impl(c, A, spec, iter0, nullptr, nullptr, packs, nullptr));
  IHS_TRY(allreduce(packs, m * d));
  IHS_TRY(gram_side_impl(c, packs, m, d, 1.0, H));
  for (int32_t t = 0; t < T; ++t) {
    const int cur = t & 1, nxt = cur ^ 1;
    const bool more = t + 1 < T;
    double *SAn = packs + nxt * pk, *gn = SAn + m * d;
    const double *x = xh + (int64_t)t * d;
    IHS_TRY(sketch_grad_impl(c, A, spec, iter0 + (uint64_t)t + 1, b, x, more ? SAn : nullptr, gn));
    IHS_TRY(more ? allreduce(SAn, pk) : allreduce(gn, d));
    if (prox < 0) {  // OLS with the Gram-only look-ahead (d > 256: the CG / Cholesky update)
      // the update first, then the Gram of S^{t+1} A: it runs beside the next
      // pass's L2-bound reductions, not beside the cooperative CG (which it
      // slowed 0.155 -> 0.22 ms, C3)
      IHS_TRY(ols_impl(c, H + cur * d * d, gn, d, x, xh + (int64_t)(t + 1) * d));
      if (more) IHS_TRY(gram_side_impl(c, SAn, m, d, 1.0, H + nxt * d * d));
    } else {
      if (more) IHS_TRY(gram_side_impl(c, SAn, m, d, 1.0, H + nxt * d * d));
      IHS_TRY(l1_impl(c, H + cur * d * d, gn, d, x, radius, cfg, xh + (int64_t)(t + 1) * d, inner_dev + t, prox));
    }
  }
  return IHS_OK;
}

// The look-ahead schedule pays when a pass over A is long next to the Gram +
// Cholesky it hides: dense, d <= 128, n d >= 2^27 (per rank: a pass of >= ~0.17 ms
// next to a ~0.11 ms factor, so also at C2 on 4 GPUs, not on 8), T >= 3, and a
// CountSketch (an SJLT pass is s gathers, next to which the d x d work is
// < 0.3% on C5 and the measured difference was within run-to-run noise).
// IHS_LOOKAHEAD=0 disables it, =1 uses it whenever supported.
// `rows` is the same on every rank (rows_for_schedule), so every rank takes the
// same schedule and issues the same collectives.
bool use_lookahead(ihs_ctx c, const ihs_matrix *A, int64_t rows, const ihs_sketch_spec *spec, int32_t T) {
  const int64_t d = A->n_cols;
  const bool ok = A->layout == IHS_DENSE_ROW_MAJOR && gram_ols_supported(d) && spec->m >= 1 && T >= 1;
  if (c->lookahead >= 0) return ok && c->lookahead != 0;
  return ok && spec->s == 1 && T >= 3 && rows * d >= (int64_t(1) << 27);
}

// l1 / LASSO look-ahead (the Gram only): dense CountSketch, n d >= 2^27, T >= 3;
// the lookahead option (IHS_LOOKAHEAD=0 / 1) as for OLS.
bool use_lookahead_pg(ihs_ctx c, const ihs_matrix *A, int64_t rows, const ihs_sketch_spec *spec, int32_t T) {
  const bool ok = A->layout == IHS_DENSE_ROW_MAJOR && spec->m >= 1 && T >= 1 && pg_supported(A->n_cols);
  if (c->lookahead >= 0) return ok && c->lookahead != 0;
  return ok && spec->s == 1 && T >= 3 && rows * A->n_cols >= (int64_t(1) << 27);
}

// a3: in-place sum over the ctx communicator (no-op on one rank).
ihs_status allreduce_impl(ihs_ctx c, double *buf, int64_t count) {
  if (!distributed(c) || count == 0) return IHS_OK;
  if (!c->comm || !load_nccl()) return IHS_ERR_COMM;
  if (g_nccl.AllReduce(buf, buf, (size_t)count, kNcclFloat64, kNcclSum, c->comm, c->stream) != 0) return IHS_ERR_COMM;
  return IHS_OK;
}

// OLS with d > 256 (a CG / Cholesky update, e.g. C3): only the Gram looks
// ahead, when it is long (m d^2 >= 2^32 multiply-adds: C3 0.30 ms).  Measured
// on C3: 0.776 -> 0.699 ms/step (the Gram beside the CG and the next CSR pass).
bool use_lookahead_gram_ols(ihs_ctx c, const ihs_matrix *A, const ihs_sketch_spec *spec, int32_t T) {
  const int64_t d = A->n_cols;
  const bool ok = d > 256 && spec->m >= 1 && T >= 1 && ols_large_supported(d);
  if (c->lookahead >= 0) return ok && c->lookahead != 0;
  return ok && T >= 3 && (double)spec->m * (double)d * (double)d >= 4294967296.0;
}

// Rows per rank that the schedule decision uses: the local count on one rank;
// with a communicator ceil(n_global / world), n_global summed over the ranks
// (shard sizes may differ by a row, and a per-rank rule could then split the
// ranks between two schedules with different collectives).
ihs_status rows_for_schedule(ihs_ctx c, int64_t n_local, int64_t *rows) {
  *rows = n_local;
  if (!distributed(c)) return IHS_OK;
  if (!c->comm || !load_nccl()) return IHS_ERR_COMM;
  double *buf;
  IHS_TRY(scratch(c, S_ROWS, 8, &buf));
  const double v = (double)n_local;
  IHS_CUDA(cudaMemcpyAsync(buf, &v, 8, cudaMemcpyHostToDevice, c->stream));
  if (g_nccl.AllReduce(buf, buf, 1, kNcclFloat64, kNcclSum, c->comm, c->stream) != 0) return IHS_ERR_COMM;
  double tot = 0.0;
  IHS_CUDA(cudaMemcpyAsync(&tot, buf, 8, cudaMemcpyDeviceToHost, c->stream));
  IHS_CUDA(cudaStreamSynchronize(c->stream));
  const int64_t ng = (int64_t)tot;
  *rows = (ng + c->world - 1) / c->world;
  return IHS_OK;
}

// Shared IHS loop (a1-a7).  constraint 0 = OLS, 1 = l1 ball.
ihs_status solve_impl(ihs_ctx c, int constraint, const ihs_matrix *A_in, const double *b_in, double radius,
                      const ihs_sketch_spec *spec, int32_t T, uint64_t iter0, const ihs_inner_cfg *cfg,
                      const double *x0_in, double *x_out, double *xh_out, ihs_iter_record *trace) {
  IHS_TRY(check_matrix(A_in));
  IHS_TRY(check_spec(spec));
  if (T < 0 || !b_in || !x_out) return IHS_ERR_INVALID_ARGUMENT;
  if (constraint >= 1 && !(radius >= 0.0)) return IHS_ERR_INVALID_ARGUMENT;
  const int64_t n = A_in->n_rows, d = A_in->n_cols, m = spec->m;
  cudaStream_t st = c->stream;
  ihs_matrix A = *A_in;
  bool any_host = false;
  // host inputs are staged into ctx buffers inside the call (e2e path)
  if (A.layout == IHS_DENSE_ROW_MAJOR && n > 0 && is_host_ptr(A.values)) {
    double *dv;
    IHS_TRY(scratch(c, S_A, (size_t)n * d * 8, &dv));
    IHS_CUDA(cudaMemcpyAsync(dv, A.values, (size_t)n * d * 8, cudaMemcpyHostToDevice, st));
    A.values = dv;
    any_host = true;
  }
  if (A.layout == IHS_CSR && is_host_ptr(A.row_ptr)) {
    int64_t *rp;
    IHS_TRY(scratch(c, S_RP, (size_t)(n + 1) * 8, &rp));
    IHS_CUDA(cudaMemcpyAsync(rp, A.row_ptr, (size_t)(n + 1) * 8, cudaMemcpyHostToDevice, st));
    A.row_ptr = rp;
    if (A.nnz > 0) {
      int32_t *cl;
      double *vl;
      IHS_TRY(scratch(c, S_COL, (size_t)A.nnz * 4, &cl));
      IHS_TRY(scratch(c, S_A, (size_t)A.nnz * 8, &vl));
      IHS_CUDA(cudaMemcpyAsync(cl, A.col_idx, (size_t)A.nnz * 4, cudaMemcpyHostToDevice, st));
      IHS_CUDA(cudaMemcpyAsync(vl, A.values, (size_t)A.nnz * 8, cudaMemcpyHostToDevice, st));
      A.col_idx = cl;
      A.values = vl;
    }
    any_host = true;
  }
  const double *b = b_in;
  if (is_host_ptr(b_in)) {
    double *db;
    IHS_TRY(scratch(c, S_B, (size_t)std::max<int64_t>(n, 1) * 8, &db));
    if (n > 0) IHS_CUDA(cudaMemcpyAsync(db, b_in, (size_t)n * 8, cudaMemcpyHostToDevice, st));
    b = db;
    any_host = true;
  }
  // packed [SA | g], H, iterate history (device)
  double *pack, *H, *xh;
  IHS_TRY(scratch(c, S_PACK, (size_t)(m * d + d) * 8, &pack));
  IHS_TRY(scratch(c, S_H, (size_t)d * d * 8, &H));
  const bool xh_host = xh_out && is_host_ptr(xh_out);
  const bool x_host = is_host_ptr(x_out);
  if (xh_out && !xh_host) {
    xh = xh_out;
  } else {
    IHS_TRY(scratch(c, S_XH, (size_t)(T + 1) * d * 8, &xh));
  }
  int32_t *inner_dev = nullptr;
  if (constraint >= 1) IHS_TRY(scratch(c, S_MISC, (size_t)std::max(T, 1) * 4, &inner_dev));
  if (x0_in) {
    IHS_CUDA(cudaMemcpyAsync(xh, x0_in, (size_t)d * 8, is_host_ptr(x0_in) ? cudaMemcpyHostToDevice
                                                                           : cudaMemcpyDeviceToDevice, st));
  } else {
    IHS_CUDA(cudaMemsetAsync(xh, 0, (size_t)d * 8, st));
  }
  double *SA = pack, *g = pack + m * d;
  const double scale = 1.0;  // SA leaves sketch_grad_impl already scaled by 1/sqrt(s)
  cudaEvent_t ev[5] = {};
  if (trace)
    for (auto &e : ev) IHS_CUDA(cudaEventCreate(&e));
  ihs_status result = IHS_OK;
  int64_t rows = n;
  if (!trace) IHS_TRY(rows_for_schedule(c, n, &rows));
  const bool lookahead =
      !trace && (constraint == 0 ? use_lookahead(c, &A, rows, spec, T) : use_lookahead_pg(c, &A, rows, spec, T));
  const bool la_gram_ols = !trace && constraint == 0 && !lookahead && use_lookahead_gram_ols(c, &A, spec, T);
  if (la_gram_ols) IHS_TRY(pg_lookahead_loop(c, &A, spec, b, iter0, T, xh, 0.0, cfg, nullptr, -1));
  if (lookahead && constraint == 0) IHS_TRY(ols_lookahead_loop(c, &A, spec, b, iter0, T, xh));
  if (lookahead && constraint >= 1)
    IHS_TRY(pg_lookahead_loop(c, &A, spec, b, iter0, T, xh, radius, cfg, inner_dev, constraint == 2 ? 1 : 0));
  // a small dense OLS problem on one rank: each iteration is one launch of one
  // CTA (small_step.cu; launch latency dominates the multi-kernel path there)
  const bool small = !lookahead && !la_gram_ols && c->small_step && !distributed(c) && constraint == 0 &&
                     A.layout == IHS_DENSE_ROW_MAJOR && small_step_supported(n, d, m, spec->s);
  if (small && !trace && T > 0) {  // all T iterations in one launch (A staged once)
    Prof pr(c, IHS_K_CHOL);
    IHS_CUDA(launch_small_step(A.values, n, d, b, xh, spec->seed, iter0, T, A.row_offset, m, spec->s,
                               spec_scale(spec), xh + d, nullptr, nullptr, nullptr, c->d_status, st, lc_of(c)));
  }
  for (int32_t t = 0; small && trace && t < T; ++t) {  // trace: one launch per iteration, timed
    const double *x = xh + (int64_t)t * d;
    double *xn = xh + (int64_t)(t + 1) * d;
    cudaEventRecord(ev[0], st);
    {
      Prof pr(c, IHS_K_CHOL);
      IHS_CUDA(launch_small_step(A.values, n, d, b, x, spec->seed, iter0 + (uint64_t)t, 1, A.row_offset, m, spec->s,
                                 spec_scale(spec), xn, nullptr, nullptr, nullptr, c->d_status, st, lc_of(c)));
    }
    if (trace) {
      cudaEventRecord(ev[1], st);
      IHS_CUDA(cudaEventSynchronize(ev[1]));
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[0], ev[1]);
      ihs_iter_record &r = trace[t];
      r.t_sketch_grad = ms;  // the whole iteration is one launch
      r.t_comm = r.t_gram = r.t_solve = 0.0;
      r.inner_iters = 0;
      ihs_status s2 = sync_status(c);
      r.status = s2;
      if (s2 != IHS_OK) {
        result = s2;
        T = t + 1;
        break;
      }
    }
  }
  for (int32_t t = 0; !lookahead && !la_gram_ols && !small && t < T; ++t) {
    const double *x = xh + (int64_t)t * d;
    double *xn = xh + (int64_t)(t + 1) * d;
    if (trace) cudaEventRecord(ev[0], st);
    IHS_TRY(sketch_grad_impl(c, &A, spec, iter0 + (uint64_t)t, b, x, SA, g));
    if (trace) cudaEventRecord(ev[1], st);
    if (distributed(c)) {
      if (!c->comm || !load_nccl()) return IHS_ERR_COMM;
      if (g_nccl.AllReduce(pack, pack, (size_t)(m * d + d), kNcclFloat64, kNcclSum, c->comm, st) != 0)
        return IHS_ERR_COMM;
    }
    if (trace) cudaEventRecord(ev[2], st);
    if (constraint == 0) {
      if (trace) cudaEventRecord(ev[3], st);  // a4 + a6 are one fused launch for d <= 128
      IHS_TRY(gram_ols_impl(c, SA, m, d, scale, g, x, xn, H));
    } else {
      IHS_TRY(gram_impl(c, SA, m, d, scale, H));
      if (trace) cudaEventRecord(ev[3], st);
      IHS_TRY(l1_impl(c, H, g, d, x, radius, cfg, xn, inner_dev + t, constraint == 2 ? 1 : 0));
    }
    if (trace) {
      cudaEventRecord(ev[4], st);
      IHS_CUDA(cudaEventSynchronize(ev[4]));
      float ms[4];
      for (int k = 0; k < 4; ++k) cudaEventElapsedTime(&ms[k], ev[k], ev[k + 1]);
      ihs_iter_record &r = trace[t];
      r.t_sketch_grad = ms[0];
      r.t_comm = ms[1];
      r.t_gram = ms[2];
      r.t_solve = ms[3];
      r.inner_iters = 0;
      if (constraint >= 1) cudaMemcpy(&r.inner_iters, inner_dev + t, 4, cudaMemcpyDeviceToHost);
      ihs_status s = sync_status(c);
      r.status = s;
      if (s == IHS_ERR_NOT_SPD || (s != IHS_OK && s != IHS_ERR_NOT_CONVERGED)) {
        result = s;
        T = t + 1;
        break;
      }
      if (s == IHS_ERR_NOT_CONVERGED) result = s;
    }
  }
  if (trace)
    for (auto &e : ev) cudaEventDestroy(e);
  const double *xlast = xh + (int64_t)T * d;
  if (x_host) {
    IHS_CUDA(cudaMemcpyAsync(x_out, xlast, (size_t)d * 8, cudaMemcpyDeviceToHost, st));
  } else if (x_out != xlast) {
    IHS_CUDA(cudaMemcpyAsync(x_out, xlast, (size_t)d * 8, cudaMemcpyDeviceToDevice, st));
  }
  if (xh_out && xh_host)
    IHS_CUDA(cudaMemcpyAsync(xh_out, xh, (size_t)(T + 1) * d * 8, cudaMemcpyDeviceToHost, st));
  if (any_host || x_host || xh_host || trace) {
    ihs_status s = sync_status(c);
    if (result == IHS_OK) result = s;
  }
  return result;
}
}  // namespace

extern "C" {

int ihs_abi_version(void) { return IHS_ABI_VERSION; }

const char *ihs_status_string(ihs_status s) {
  switch (s) {
    case IHS_OK: return "ok";
    case IHS_ERR_INVALID_ARGUMENT: return "invalid argument";
    case IHS_ERR_DIMENSION_MISMATCH: return "dimension mismatch";
    case IHS_ERR_NOT_SPD: return "Hessian sketch not positive definite";
    case IHS_ERR_NOT_CONVERGED: return "inner solver did not converge";
    case IHS_ERR_CUDA: return "CUDA error";
    case IHS_ERR_COMM: return "communication error";
    case IHS_ERR_OUT_OF_MEMORY: return "out of device memory";
    case IHS_ERR_UNSUPPORTED: return "unsupported shape";
  }
  return "unknown status";
}

ihs_status ihs_ctx_create(ihs_ctx *out, int device, void *stream) {
  if (!out) return IHS_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
    cudaGetLastError();
    return IHS_ERR_CUDA;
  }
  DevGuard g(device);
  ihs_ctx c = new ihs_ctx_s();
  c->device = device;
  c->stream = (cudaStream_t)stream;
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (cudaMalloc(&c->d_status, 4 * sizeof(int)) != cudaSuccess) {  // [0] status, [1] reduce counter
    delete c;
    return IHS_ERR_OUT_OF_MEMORY;
  }
  cudaMemset(c->d_status, 0, 4 * sizeof(int));
  // initial option values from the environment (ihs_ctx_set_option changes them per ctx)
  if (const char *e = getenv("IHS_PREFETCH")) c->prefetch = std::strcmp(e, "0") != 0;
  if (const char *e = getenv("IHS_SJLT")) c->sjlt_onepass = !std::strcmp(e, "passes") ? 0 : !std::strcmp(e, "gradpass") ? 2 : 1;
  if (const char *e = getenv("IHS_LOOKAHEAD")) c->lookahead = std::strcmp(e, "0") != 0 ? 1 : 0;
  if (const char *e = getenv("IHS_OLS")) c->ols_large = !std::strcmp(e, "chol") ? 2 : !std::strcmp(e, "cg") ? 0 : 1;
  if (const char *e = getenv("IHS_FUSE")) c->fuse_max_d = !std::strcmp(e, "0") ? 0 : 128;
  if (const char *e = getenv("IHS_PG_WARM")) c->pg_warm = std::strcmp(e, "0") != 0;
  if (const char *e = getenv("IHS_PG_CLUSTER")) c->pg_cluster = atoi(e);
  *out = c;
  return IHS_OK;
}

ihs_status ihs_ctx_destroy(ihs_ctx c) {
  if (!c) return IHS_ERR_INVALID_ARGUMENT;
  DevGuard g(c->device);
  join_factor(c);
  cudaStreamSynchronize(c->stream);
  if (c->fstream) {
    cudaStreamSynchronize(c->fstream);
    cudaStreamDestroy(c->fstream);
    cudaEventDestroy(c->ev_fmain);
    for (auto &f : c->fac) cudaEventDestroy(f.done);
  }
  if (c->side) {
    cudaStreamSynchronize(c->side);
    cudaStreamDestroy(c->side);
    cudaEventDestroy(c->ev_side);
    cudaEventDestroy(c->ev_main);
  }
  for (int s = 0; s < S_NSLOTS; ++s)
    if (c->slot[s]) cudaFree(c->slot[s]);
  if (c->d_status) cudaFree(c->d_status);
  if (c->d_L) cudaFree(c->d_L);
  if (c->ev_switch) cudaEventDestroy(c->ev_switch);
  if (c->comm && g_nccl.loaded) g_nccl.CommDestroy(c->comm);
  for (cudaEvent_t e : c->pool) cudaEventDestroy(e);
  delete c;
  return IHS_OK;
}

ihs_status ihs_ctx_set_stream(ihs_ctx c, void *stream) {
  if (!c) return IHS_ERR_INVALID_ARGUMENT;
  // pending factor / side work stays pending: it is joined into whichever stream
  // the ctx is bound to when a call needs it (wait_factor / join_side).  Work
  // already enqueued on the old stream is ordered before the new one (the ctx
  // scratch, status word and reduction counter are shared by both).
  cudaStream_t ns = (cudaStream_t)stream;
  if (ns != c->stream) {
    DevGuard g(c->device);
    if (!c->ev_switch) IHS_CUDA(cudaEventCreateWithFlags(&c->ev_switch, cudaEventDisableTiming));
    IHS_CUDA(cudaEventRecord(c->ev_switch, c->stream));
    IHS_CUDA(cudaStreamWaitEvent(ns, c->ev_switch, 0));
    c->stream = ns;
  }
  return IHS_OK;
}

ihs_status ihs_ctx_synchronize(ihs_ctx c) {
  if (!c) return IHS_ERR_INVALID_ARGUMENT;
  DevGuard g(c->device);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return from_cuda(e);
  return sync_status(c);
}

int64_t ihs_ctx_kernel_launches(ihs_ctx c) { return c ? c->launches : -1; }

namespace {
struct OptionDef {
  const char *name;
  int ihs_ctx_s::*field;
  int lo, hi;
};
const OptionDef kOptions[] = {
    {"lookahead", &ihs_ctx_s::lookahead, -1, 1},   {"sjlt_onepass", &ihs_ctx_s::sjlt_onepass, 0, 2},
    {"ols_large", &ihs_ctx_s::ols_large, 0, 2},    {"fuse_max_d", &ihs_ctx_s::fuse_max_d, 0, 128},
    {"pg_warm", &ihs_ctx_s::pg_warm, 0, 1},       {"small_step", &ihs_ctx_s::small_step, 0, 1},
    {"pg_cluster", &ihs_ctx_s::pg_cluster, 0, 16}, {"la_gram_sms", &ihs_ctx_s::la_gram_sms, 0, 1024},
    {"la_gram_tile", &ihs_ctx_s::la_gram_tile, 0, 128},
};
}  // namespace

ihs_status ihs_ctx_set_option(ihs_ctx c, const char *name, int64_t value) {
  if (!c || !name) return IHS_ERR_INVALID_ARGUMENT;
  if (!std::strcmp(name, "prefetch")) {
    if (value < 0 || value > 1) return IHS_ERR_INVALID_ARGUMENT;
    c->prefetch = value != 0;
    return IHS_OK;
  }
  for (const OptionDef &o : kOptions)
    if (!std::strcmp(name, o.name)) {
      if (value < o.lo || value > o.hi) return IHS_ERR_INVALID_ARGUMENT;
      c->*(o.field) = (int)value;
      return IHS_OK;
    }
  return IHS_ERR_INVALID_ARGUMENT;
}

ihs_status ihs_ctx_get_option(ihs_ctx c, const char *name, int64_t *value) {
  if (!c || !name || !value) return IHS_ERR_INVALID_ARGUMENT;
  if (!std::strcmp(name, "prefetch")) {
    *value = c->prefetch ? 1 : 0;
    return IHS_OK;
  }
  for (const OptionDef &o : kOptions)
    if (!std::strcmp(name, o.name)) {
      *value = c->*(o.field);
      return IHS_OK;
    }
  return IHS_ERR_INVALID_ARGUMENT;
}

ihs_status ihs_ctx_set_profiling(ihs_ctx c, int enable) {
  if (!c) return IHS_ERR_INVALID_ARGUMENT;
  c->profiling = enable != 0;
  return IHS_OK;
}

ihs_status ihs_ctx_profile(ihs_ctx c, int group, double *total_ms, int64_t *launches) {
  if (!c || group < 0 || group >= IHS_K_COUNT || !total_ms || !launches) return IHS_ERR_INVALID_ARGUMENT;
  DevGuard g(c->device);
  IHS_CUDA(cudaStreamSynchronize(c->stream));
  double tot = 0.0;
  int64_t k = 0;
  for (auto &r : c->recs)
    if (r.group == group) {
      float ms = 0.f;
      IHS_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
      tot += ms;
      ++k;
    }
  *total_ms = tot;
  *launches = k;
  return IHS_OK;
}

ihs_status ihs_ctx_profile_reset(ihs_ctx c) {
  if (!c) return IHS_ERR_INVALID_ARGUMENT;
  DevGuard g(c->device);
  IHS_CUDA(cudaStreamSynchronize(c->stream));
  c->recs.clear();
  c->pool_used = 0;
  return IHS_OK;
}

ihs_status ihs_nccl_unique_id(void *out128) {
  if (!out128) return IHS_ERR_INVALID_ARGUMENT;
  if (!load_nccl()) return IHS_ERR_COMM;
  nccl_uid id;
  if (g_nccl.GetUniqueId(&id) != 0) return IHS_ERR_COMM;
  std::memcpy(out128, &id, sizeof(id));
  return IHS_OK;
}

ihs_status ihs_ctx_set_comm(ihs_ctx c, int rank, int world, const void *uid) {
  if (!c || world < 1 || rank < 0 || rank >= world || c->comm) return IHS_ERR_INVALID_ARGUMENT;
  c->rank = rank;
  c->world = world;
  if (world == 1 && !uid) return IHS_OK;  // no communicator: the single-rank schedules
  if (!uid) return IHS_ERR_INVALID_ARGUMENT;
  if (!load_nccl()) return IHS_ERR_COMM;
  DevGuard g(c->device);
  nccl_uid id;
  std::memcpy(&id, uid, sizeof(id));
  if (g_nccl.CommInitRank(&c->comm, world, id, rank) != 0) return IHS_ERR_COMM;
  return IHS_OK;
}

ihs_status ihs_allreduce_sum(ihs_ctx c, double *buf, int64_t count) {
  if (!c || (!buf && count > 0) || count < 0) return IHS_ERR_INVALID_ARGUMENT;
  DevGuard g(c->device);
  return allreduce_impl(c, buf, count);
}

ihs_status ihs_allreduce_multimem(ihs_ctx c, double *mc_buf, uint32_t *const *signal_pads, int rank, int world,
                                  int64_t count, int64_t pad_slots) {
  if (!c || count < 0 || world < 1 || rank < 0 || rank >= world) return IHS_ERR_INVALID_ARGUMENT;
  if (count == 0) return IHS_OK;
  if (!mc_buf || !signal_pads) return IHS_ERR_INVALID_ARGUMENT;
  DevGuard g(c->device);
  const int blocks = nvls_blocks(count, world, c->num_sms);
  if ((int64_t)blocks * world > pad_slots) return IHS_ERR_UNSUPPORTED;
  IHS_CUDA(launch_nvls_allreduce(mc_buf, signal_pads, rank, world, count, blocks, c->stream, lc_of(c)));
  return IHS_OK;
}

ihs_status ihs_hash(ihs_ctx c, const ihs_sketch_spec *spec, uint64_t iter, int64_t row_begin, int64_t count,
                    int32_t *bucket, int8_t *sign) {
  if (!c) return IHS_ERR_INVALID_ARGUMENT;
  IHS_TRY(check_spec(spec));
  if (row_begin < 0 || count < 0 || (count > 0 && (!bucket || !sign))) return IHS_ERR_INVALID_ARGUMENT;
  DevGuard g(c->device);
  IHS_CUDA(launch_hash_export(iter_key(spec->seed, iter), (uint32_t)spec->s, (uint32_t)(spec->m / spec->s), row_begin,
                              count, bucket, sign, c->stream, lc_of(c)));
  return IHS_OK;
}

ihs_status ihs_sketch(ihs_ctx c, const ihs_matrix *A, const ihs_sketch_spec *spec, uint64_t iter, double *SA,
                      int reduce) {
  if (!c || !SA) return IHS_ERR_INVALID_ARGUMENT;
  IHS_TRY(check_matrix(A));
  IHS_TRY(check_spec(spec));
  DevGuard g(c->device);
  IHS_TRY(sketch_grad_impl(c, A, spec, iter, nullptr, nullptr, SA, nullptr));
  return reduce ? allreduce_impl(c, SA, spec->m * A->n_cols) : IHS_OK;
}

ihs_status ihs_grad(ihs_ctx c, const ihs_matrix *A, const double *b, const double *x, double *gout, int reduce) {
  if (!c || !gout || !x || (!b && A && A->n_rows > 0)) return IHS_ERR_INVALID_ARGUMENT;
  IHS_TRY(check_matrix(A));
  DevGuard g(c->device);
  ihs_sketch_spec dummy{IHS_COUNTSKETCH, 1, 1, 0};
  IHS_TRY(sketch_grad_impl(c, A, &dummy, 0, b, x, nullptr, gout));
  return reduce ? allreduce_impl(c, gout, A->n_cols) : IHS_OK;
}

ihs_status ihs_sketch_grad(ihs_ctx c, const ihs_matrix *A, const ihs_sketch_spec *spec, uint64_t iter, const double *b,
                           const double *x, double *SA, double *gout, int reduce) {
  if (!c || !SA || !gout || !x || (!b && A && A->n_rows > 0)) return IHS_ERR_INVALID_ARGUMENT;
  IHS_TRY(check_matrix(A));
  IHS_TRY(check_spec(spec));
  DevGuard g(c->device);
  IHS_TRY(sketch_grad_impl(c, A, spec, iter, b, x, SA, gout));
  if (!reduce) return IHS_OK;
  const int64_t md = spec->m * A->n_cols;
  if (gout == SA + md) return allreduce_impl(c, SA, md + A->n_cols);  // packed [SA | g]: one all-reduce
  IHS_TRY(allreduce_impl(c, SA, md));
  return allreduce_impl(c, gout, A->n_cols);
}

ihs_status ihs_ols_lookahead_step(ihs_ctx c, const ihs_matrix *A, const ihs_sketch_spec *spec, uint64_t iter_next,
                                  const double *b, const double *x, const double *Hinv, double *SA_next,
                                  double *Hinv_next, double *gout, double *xn) {
  if (!c || !x || !Hinv || !gout || !xn || (!b && A && A->n_rows > 0) || (Hinv_next && !SA_next))
    return IHS_ERR_INVALID_ARGUMENT;
  IHS_TRY(check_matrix(A));
  IHS_TRY(check_spec(spec));
  if (A->layout != IHS_DENSE_ROW_MAJOR || A->n_cols > 1024) return IHS_ERR_UNSUPPORTED;
  if (Hinv_next && !gram_ols_supported(A->n_cols)) return IHS_ERR_UNSUPPORTED;
  DevGuard g(c->device);
  const LookStep ls{Hinv, x, xn, Hinv_next};
  return sketch_grad_impl(c, A, spec, iter_next, b, x, SA_next, gout, &ls);
}

ihs_status ihs_small_step(ihs_ctx c, const ihs_matrix *A, const double *b, const ihs_sketch_spec *spec, uint64_t iter,
                          const double *x, double *xn, double *SA_out, double *g_out, double *H_out) {
  if (!c || !x || !xn || (!b && A && A->n_rows > 0)) return IHS_ERR_INVALID_ARGUMENT;
  IHS_TRY(check_matrix(A));
  IHS_TRY(check_spec(spec));
  if (A->layout != IHS_DENSE_ROW_MAJOR || !small_step_supported(A->n_rows, A->n_cols, spec->m, spec->s))
    return IHS_ERR_UNSUPPORTED;
  DevGuard g(c->device);
  Prof pr(c, IHS_K_CHOL);
  IHS_CUDA(launch_small_step(A->values, A->n_rows, A->n_cols, b, x, spec->seed, iter, 1, A->row_offset, spec->m,
                             spec->s, spec_scale(spec), xn, SA_out, g_out, H_out, c->d_status, c->stream, lc_of(c)));
  return IHS_OK;
}

ihs_status ihs_gram(ihs_ctx c, const double *SA, int64_t m, int64_t d, double scale, double *H) {
  if (!c || !SA || !H || m < 1 || d < 1 || !std::isfinite(scale)) return IHS_ERR_INVALID_ARGUMENT;
  DevGuard g(c->device);
  return gram_impl(c, SA, m, d, scale, H);
}

ihs_status ihs_gram_ols_update(ihs_ctx c, const double *SA, int64_t m, int64_t d, double scale, const double *gv,
                               const double *x, double *xn, double *H) {
  if (!c || !SA || !gv || !x || !xn || !H || d < 1 || m < 0) return IHS_ERR_INVALID_ARGUMENT;
  DevGuard g(c->device);
  return gram_ols_impl(c, SA, m, d, scale, gv, x, xn, H);
}

ihs_status ihs_ols_factor(ihs_ctx c, const double *SA, int64_t m, int64_t d, double scale, double *Hinv) {
  if (!c || !SA || !Hinv || m < 1 || d < 1 || !std::isfinite(scale)) return IHS_ERR_INVALID_ARGUMENT;
  DevGuard g(c->device);
  return ols_factor_impl(c, SA, m, d, scale, Hinv);
}

ihs_status ihs_gram_lookahead(ihs_ctx c, const double *SA, int64_t m, int64_t d, double scale, double *H) {
  if (!c || !SA || !H || m < 1 || d < 1 || !std::isfinite(scale)) return IHS_ERR_INVALID_ARGUMENT;
  DevGuard g(c->device);
  return gram_side_impl(c, SA, m, d, scale, H);
}

ihs_status ihs_ols_apply(ihs_ctx c, const double *Hinv, const double *gv, int64_t d, const double *x, double *xn) {
  if (!c || !Hinv || !gv || !x || !xn || d < 1) return IHS_ERR_INVALID_ARGUMENT;
  if (d > 1024) return IHS_ERR_UNSUPPORTED;
  DevGuard g(c->device);
  return ols_apply_impl(c, Hinv, gv, d, x, xn);
}

ihs_status ihs_ols_update(ihs_ctx c, const double *H, const double *gv, int64_t d, const double *x, double *xn) {
  if (!c || !H || !gv || !x || !xn || d < 1) return IHS_ERR_INVALID_ARGUMENT;
  DevGuard g(c->device);
  return ols_impl(c, H, gv, d, x, xn);
}

ihs_status ihs_l1ball_update(ihs_ctx c, const double *H, const double *gv, int64_t d, const double *x, double radius,
                             const ihs_inner_cfg *cfg, double *xn, int32_t *inner) {
  if (!c || !H || !gv || !x || !xn || d < 1 || !(radius >= 0.0)) return IHS_ERR_INVALID_ARGUMENT;
  DevGuard g(c->device);
  return l1_impl(c, H, gv, d, x, radius, cfg, xn, inner);
}

ihs_status ihs_lasso_update(ihs_ctx c, const double *H, const double *gv, int64_t d, const double *x, double lambda,
                            const ihs_inner_cfg *cfg, double *xn, int32_t *inner) {
  if (!c || !H || !gv || !x || !xn || d < 1 || !(lambda >= 0.0)) return IHS_ERR_INVALID_ARGUMENT;
  DevGuard g(c->device);
  return l1_impl(c, H, gv, d, x, lambda, cfg, xn, inner, 1);
}

ihs_status ihs_solve_lasso(ihs_ctx c, const ihs_matrix *A, const double *b, double lambda,
                           const ihs_sketch_spec *spec, int32_t n_iters, uint64_t iter0, const ihs_inner_cfg *cfg,
                           const double *x0, double *x, double *x_hist, ihs_iter_record *trace) {
  if (!c) return IHS_ERR_INVALID_ARGUMENT;
  DevGuard g(c->device);
  return solve_impl(c, 2, A, b, lambda, spec, n_iters, iter0, cfg, x0, x, x_hist, trace);
}

ihs_status ihs_solve_ols(ihs_ctx c, const ihs_matrix *A, const double *b, const ihs_sketch_spec *spec, int32_t n_iters,
                         uint64_t iter0, const double *x0, double *x, double *x_hist, ihs_iter_record *trace) {
  if (!c) return IHS_ERR_INVALID_ARGUMENT;
  DevGuard g(c->device);
  return solve_impl(c, 0, A, b, 0.0, spec, n_iters, iter0, nullptr, x0, x, x_hist, trace);
}

ihs_status ihs_solve_l1ball(ihs_ctx c, const ihs_matrix *A, const double *b, double radius,
                            const ihs_sketch_spec *spec, int32_t n_iters, uint64_t iter0, const ihs_inner_cfg *cfg,
                            const double *x0, double *x, double *x_hist, ihs_iter_record *trace) {
  if (!c) return IHS_ERR_INVALID_ARGUMENT;
  DevGuard g(c->device);
  return solve_impl(c, 1, A, b, radius, spec, n_iters, iter0, cfg, x0, x, x_hist, trace);
}

ihs_status ihs_pred_err2(ihs_ctx c, const ihs_matrix *A, const double *X, int32_t count, const double *xref,
                         double *err2, double *ref2) {
  if (!c || !xref || !err2 || !ref2 || count < 0 || (count > 0 && !X)) return IHS_ERR_INVALID_ARGUMENT;
  IHS_TRY(check_matrix(A));
  if (A->layout == IHS_DENSE_ROW_MAJOR && A->n_cols > 1024) return IHS_ERR_UNSUPPORTED;
  DevGuard g(c->device);
  const int64_t d = A->n_cols;
  const int64_t nb = grad_dense_blocks(A->n_rows, d, c->num_sms);
  double *sc, *acc;
  IHS_TRY(scratch(c, S_ERR, (size_t)(((d + 31) / 32) * 32 + nb) * 8, &sc));
  IHS_TRY(scratch(c, S_MISC, (size_t)(count + 1) * 8, &acc));
  IHS_CUDA(launch_pred_err2_impl(A->layout, A->n_rows, d, A->values, A->row_ptr, A->col_idx, X, count, xref, acc, sc,
                                 c->num_sms, c->stream, lc_of(c)));
  if (count > 0) IHS_CUDA(cudaMemcpyAsync(err2, acc, (size_t)count * 8, cudaMemcpyDeviceToDevice, c->stream));
  IHS_CUDA(cudaMemcpyAsync(ref2, acc + count, 8, cudaMemcpyDeviceToDevice, c->stream));
  return IHS_OK;
}

}  // extern "C"
