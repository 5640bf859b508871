/*
 * include/ihs.h -- C ABI of the B200-native Iterative Hessian Sketch hot path
 * (arXiv 1910.14166, /root/reference/PAPER.md).  Implemented by
 * paper_1910_14166_b200/libihs.so (hand-written sm_100a CUDA).
 *
 * Conventions (apply to every call unless its comment says otherwise)
 *  - Arrays are fp64 / int row-major, DEVICE pointers on the ctx's device, owned
 *    by the caller.  The library owns only the scratch inside an ihs_ctx.
 *  - Every call is stream-ordered on the ctx stream and returns as soon as its
 *    kernels are enqueued.  Argument errors are returned synchronously and
 *    nothing is enqueued.  Asynchronous CUDA faults and device-side statuses
 *    (a non-positive Cholesky pivot, an inner solver hitting its cap) surface
 *    at the next ihs_ctx_synchronize().  The library never aborts or prints.
 *  - "Global row": rank k of P holds rows [row_offset, row_offset+n_rows) of
 *    the global A; the sketch hash always uses the global row index, so the
 *    per-rank partial sketches sum to S A exactly (linearity).
 *  - Hash (reading R1; BASELINE.json north_star): with
 *    SM(x) = splitmix64 finaliser of x + 0x9E3779B97F4A7C15,
 *    k_t = SM(SM(seed) ^ t), w = SM(k_t ^ (i*s + j)) for global row i and
 *    SJLT block j, M = m/s, bucket = j*M + ((w>>32)*M >> 32),
 *    sign = (w & 1) ? -1 : +1.
 *  - Sign of the gradient (reading R21): g = +A^T (b - A x) = -grad f.
 */
#ifndef IHS_H
#define IHS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IHS_ABI_VERSION 2

typedef enum {
    IHS_OK = 0,
    IHS_ERR_INVALID_ARGUMENT = 1,   /* null pointer, negative size, bad spec */
    IHS_ERR_DIMENSION_MISMATCH = 2, /* e.g. m not divisible by s */
    IHS_ERR_NOT_SPD = 3,            /* H not positive definite: Cholesky pivot <= 0, or (CG path,
                                       d > 160) a non-positive diagonal / curvature p.Hp <= 0 (R13, R22) */
    IHS_ERR_NOT_CONVERGED = 4,      /* inner PG hit max_inner (best iterate written), or the
                                       OLS CG hit its cap (x_next = x + last u) */
    IHS_ERR_CUDA = 5,               /* CUDA runtime / launch / async fault */
    IHS_ERR_COMM = 6,               /* NCCL failure or communicator missing */
    IHS_ERR_OUT_OF_MEMORY = 7,      /* scratch allocation failed */
    IHS_ERR_UNSUPPORTED = 8         /* shape outside the kernels' limits */
} ihs_status;

/* Sketch families (section 2). */
typedef enum { IHS_COUNTSKETCH = 0, IHS_SJLT = 1 } ihs_family;

typedef struct {
    int32_t family; /* ihs_family */
    int32_t s;      /* nonzeros per column of S: 1 for CountSketch; SJLT: 1 <= s <= m, s | m */
    int64_t m;      /* sketch rows, m >= 1 (m > n is legal) */
    uint64_t seed;  /* hash seed */
} ihs_sketch_spec;

typedef enum { IHS_DENSE_ROW_MAJOR = 0, IHS_CSR = 1 } ihs_layout;

/* A local row block of A.  Dense: values[n_rows*n_cols], row-major, 16-byte
 * aligned.  CSR: row_ptr[n_rows+1] with row_ptr[0] = 0 (rebased per shard),
 * col_idx[nnz] strictly increasing within a row and < n_cols, values[nnz]. */
typedef struct {
    int32_t layout;       /* ihs_layout */
    int32_t reserved;     /* must be 0 */
    int64_t n_rows;       /* local rows, 0 <= n_rows < 2^31 */
    int64_t n_cols;       /* d >= 1 */
    int64_t row_offset;   /* global index of local row 0 */
    const double *values;
    const int64_t *row_ptr;
    const int32_t *col_idx;
    int64_t nnz;
} ihs_matrix;

/* Inner projected-gradient configuration (reading R10; SPEC.md:266 gives
 * 50 power iterations and a 5000-step cap for its own CPU solver). */
typedef struct {
    int32_t max_inner;        /* cap on PG steps per outer iteration (default 20000) */
    int32_t power_iters;      /* power iterations for lambda_max(H) from 1/sqrt(d): the first
                                 update of a context for this d (default 50) */
    double inner_tol;         /* stop when ||y+ - y|| <= tol * max(1, ||y||) (default 1e-14) */
    double lip_safety;        /* step 1/(safety * lambda_max) (default 1.05) */
    int32_t warm_power_iters; /* power iterations on later updates with the same d, started from
                                 the previous update's vector (default 12; >= 1; set it to
                                 power_iters to give every update the cold count) */
    int32_t reserved;         /* must be 0 */
} ihs_inner_cfg;

/* Per-iteration record written by the solve calls (host memory). Times in ms
 * from CUDA events on the ctx stream; filled only when trace != NULL. */
typedef struct {
    double t_sketch_grad; /* hash/sort + sketch + gradient (a1, a2, a5) */
    double t_comm;        /* allreduce of [SA | g] (a3), 0 at P = 1 */
    double t_gram;        /* (SA)^T SA (a4) */
    double t_solve;       /* inner QP (a6) */
    int32_t inner_iters;  /* PG steps (l1 ball) or 0 */
    int32_t status;       /* ihs_status of this iteration's inner solve */
} ihs_iter_record;

typedef struct ihs_ctx_s *ihs_ctx;

int ihs_abi_version(void);
const char *ihs_status_string(ihs_status st);

/* Create a context on `device` bound to `stream` (a cudaStream_t; NULL = the
 * legacy default stream).  One context per (device, stream); no global state. */
ihs_status ihs_ctx_create(ihs_ctx *out, int device, void *stream);
ihs_status ihs_ctx_destroy(ihs_ctx ctx);
/* Rebind the ctx to another stream.  Work the ctx runs on its own streams (the
 * sort prefetch, look-ahead factors) stays pending and is joined into the stream
 * bound when a later call needs its result. */
ihs_status ihs_ctx_set_stream(ihs_ctx ctx, void *stream);
/* Wait for the ctx stream; return the first asynchronous error or device-side
 * status (IHS_ERR_NOT_SPD, IHS_ERR_NOT_CONVERGED) raised since the last call,
 * and clear it. */
ihs_status ihs_ctx_synchronize(ihs_ctx ctx);
/* Number of kernels this ctx has launched so far (bench evidence). */
int64_t ihs_ctx_kernel_launches(ihs_ctx ctx);

/* Per-context options (initial values from the IHS_* environment variables
 * named in brackets, read at ihs_ctx_create).  Unknown name or out-of-range
 * value: IHS_ERR_INVALID_ARGUMENT.
 *   "lookahead"    -1 (default) look-ahead schedules of the solve calls by size,
 *                  0 off, 1 whenever supported                    [IHS_LOOKAHEAD]
 *   "sjlt_onepass" 1 (default) dense SJLT in one read of A, the gradient of
 *                  ihs_sketch_grad riding on the same pass (d <= 128); 2 the same
 *                  with the gradient in its own pass; 0 as s sorted CountSketch
 *                  passes (bit-identical to the oracle) [IHS_SJLT=passes|gradpass]
 *   "ols_large"    d > 160 OLS step: 1 (default) conjugate gradients, then the
 *                  blocked Cholesky in the same launch when CG does not finish;
 *                  0 CG only (IHS_ERR_NOT_CONVERGED at its cap); 2 the Cholesky
 *                  only (positive definiteness certified exactly, reading R22) [IHS_OLS]
 *   "fuse_max_d"   a4 + a6 in one cluster launch up to this d (0..128, default 64) [IHS_FUSE]
 *   "pg_warm"      1 (default) warm-started power iteration across l1 / LASSO updates [IHS_PG_WARM]
 *   "small_step"   1 (default) ihs_solve_ols on one rank runs each iteration of a small dense
 *                  problem (d <= 32, n <= 32768, its working set in one CTA's shared memory)
 *                  as ONE launch of one CTA; 0 the general multi-kernel path
 *   "la_gram_tile" the look-ahead Gram of d > 256 (ihs_gram_lookahead, the OLS solve with the
 *                  CG update): 0 / 64 (default) the 64 x 64-tile stream-K, whose two
 *                  128-thread CTAs per SM leave the pass's CTAs room on the same SMs;
 *                  128 the 128 x 128-tile stream-K (one 512-thread CTA holds an SM)
 *   "la_gram_sms"  SMs that Gram takes (0 default: all; >= 64): the rest stay with the pass
 *   "prefetch"     1 (default) the next iteration's sort on the side stream   [IHS_PREFETCH] */
ihs_status ihs_ctx_set_option(ihs_ctx ctx, const char *name, int64_t value);
ihs_status ihs_ctx_get_option(ihs_ctx ctx, const char *name, int64_t *value);

/* Per-kernel timing (bench evidence): when enabled, CUDA events are recorded on
 * the ctx stream around every launch of the kernel groups below.
 * ihs_ctx_profile synchronises and returns the summed elapsed ms and the
 * number of timed launches of one group since the last reset. */
typedef enum {
    IHS_K_SORT = 0,        /* a1: hash + stable counting sort (hist, scan, scatter) */
    IHS_K_SKETCH = 1,      /* a2 (+a5): bucket-ordered CountSketch gather, fused gradient */
    IHS_K_SJLT = 2,        /* a2: dense SJLT smem-tile kernel + split reduction */
    IHS_K_CSR = 3,         /* a2 + a5 on CSR */
    IHS_K_GRAD = 4,        /* a5 standalone dense gradient */
    IHS_K_REDUCE = 5,      /* fixed-order partial reductions */
    IHS_K_GRAM = 6,        /* a4 DMMA Gram + reduction */
    IHS_K_CHOL = 7,        /* a6 Cholesky update */
    IHS_K_PG = 8,          /* a6 projected gradient */
    IHS_K_FACTOR = 9,      /* look-ahead a4 + a6: Gram + Cholesky + inverse (factor stream) */
    IHS_K_APPLY = 10,      /* look-ahead a6: x + H^{-1} g */
    IHS_K_COUNT = 11
} ihs_kernel_group;
ihs_status ihs_ctx_set_profiling(ihs_ctx ctx, int enable);
ihs_status ihs_ctx_profile(ihs_ctx ctx, int group, double *total_ms, int64_t *launches);
ihs_status ihs_ctx_profile_reset(ihs_ctx ctx);

/* Multi-GPU (BASELINE.json north_star: one allreduce of [SA | g] per
 * iteration).  ihs_nccl_unique_id writes NCCL's 128-byte id (call on rank 0,
 * broadcast it); ihs_ctx_set_comm creates this rank's communicator.  NCCL is
 * resolved at run time from the libnccl.so.2 already loaded in the process.
 * world == 1 with unique_id128 == NULL: no communicator (single-rank
 * schedules); world == 1 with an id: a one-rank communicator, and the solve
 * calls take their collective schedules (NCCL all-reduces over one rank --
 * the multi-rank code path checked on one GPU).  Once per ctx: a second call
 * on a ctx that holds a communicator is IHS_ERR_INVALID_ARGUMENT;
 * IHS_ERR_COMM when NCCL cannot be loaded or the init fails. */
ihs_status ihs_nccl_unique_id(void *out128);
ihs_status ihs_ctx_set_comm(ihs_ctx ctx, int rank, int world, const void *unique_id128);
/* In-place sum of count doubles across the ctx communicator (a3). */
ihs_status ihs_allreduce_sum(ihs_ctx ctx, double *buf, int64_t count);
/* a3 over NVLink SHARP (the sum of the per-rank partial
 * sketches and gradients, exact by linearity): in-place sum of
 * count doubles of a symmetric buffer across `world` ranks, in one kernel that
 * reduces with multimem.ld_reduce.add.f64 on the buffer's multicast address
 * (`mc_buf`, device) and broadcasts with multimem.st -- rank r handles slice r
 * -- between two barriers over the ranks' signal pads (`signal_pads`: device
 * array of `world` unicast pointers, each >= pad_slots u32, zero before first
 * use and left zero).  The buffer, its multicast mapping and the pads come
 * from the caller (e.g. torch symmetric memory); every rank calls with the
 * same count.  IHS_ERR_UNSUPPORTED when the pads are too small (blocks x world
 * slots, blocks <= SM count).  Not the default exchange (NCCL is): every rank
 * receives the same broadcast value. */
ihs_status ihs_allreduce_multimem(ihs_ctx ctx, double *mc_buf, uint32_t *const *signal_pads, int rank, int world,
                                  int64_t count, int64_t pad_slots);

/* a1: export buckets/signs of global rows [row_begin, row_begin+count), arrays
 * of count*s entries ordered (row, block) -- bit-exact test interface.
 * Device pointers. */
ihs_status ihs_hash(ihs_ctx ctx, const ihs_sketch_spec *spec, uint64_t iter,
                    int64_t row_begin, int64_t count, int32_t *bucket, int8_t *sign);

/* a2: SA = S^(iter) A_local (m x d) (section 2;
 * SJLT scaled by 1/sqrt(s)).  reduce = 0: the local partial
 * sketch; reduce != 0: summed in place over the ctx communicator afterwards
 * (the full S A on every rank, by linearity -- BASELINE.json north_star; the
 * same as ihs_allreduce_sum(SA, m*d); a no-op at world size 1).
 * Dense SJLT is deterministic but, with "sjlt_onepass", not bit-identical to
 * the oracle's single ascending sum (within 1e-12, reading R3). */
ihs_status ihs_sketch(ihs_ctx ctx, const ihs_matrix *A, const ihs_sketch_spec *spec,
                      uint64_t iter, double *SA, int reduce);

/* a5: g = A_local^T (b_local - A_local x) (d) (the linear term of Eq. (2),
 * PAPER.md:83-86); reduce as for ihs_sketch. */
ihs_status ihs_grad(ihs_ctx ctx, const ihs_matrix *A, const double *b, const double *x,
                    double *g, int reduce);

/* a2 + a5 (NEXT-1): one pass over A where the layout allows (dense CountSketch
 * with even d <= 256, CSR); dense SJLT: the one-read sketch pass and the
 * gradient stream side by side; otherwise two passes.  Writes SA (m x d) and
 * g (d); g may equal SA + m*d so that [SA | g] is one packed buffer: with
 * reduce != 0 and g == SA + m*d it is summed over the communicator in ONE
 * all-reduce of m*d + d doubles (a3), otherwise SA and g separately. */
ihs_status ihs_sketch_grad(ihs_ctx ctx, const ihs_matrix *A, const ihs_sketch_spec *spec,
                           uint64_t iter, const double *b, const double *x,
                           double *SA, double *g, int reduce);

/* a4: H = (SA)^T SA (d x d, full symmetric), fp64 on the DMMA tensor pipe
 * (PAPER.md:95, 104-106).  `scale` multiplies every SA entry on load (1.0, or
 * 1/sqrt(s) for an unscaled SJLT sum). */
ihs_status ihs_gram(ihs_ctx ctx, const double *SA, int64_t m, int64_t d, double scale,
                    double *H);

/* a4 + a6 for OLS in one call: H = scale^2 SA^T SA (written to H, d x d) and
 * x_next = x + H^{-1} g.  d <= 64 (IHS_FUSE=1: d <= 128): one thread-block-
 * cluster launch (Gram partials on DMMA, reduced through distributed shared
 * memory straight into the Cholesky CTA); otherwise ihs_gram followed by
 * ihs_ols_update.  Statuses as for ihs_ols_update. */
ihs_status ihs_gram_ols_update(ihs_ctx ctx, const double *SA, int64_t m, int64_t d, double scale,
                               const double *g, const double *x, double *x_next, double *H);

/* Look-ahead OLS.  S^{t+1} does not depend on x
 * (Eq. (2): a fresh sketch per iteration, hashed from
 * (seed, iteration, row) -- reading R1), so H_{t+1} = (S^{t+1}A)^T S^{t+1}A can
 * be formed and factorised while the pass over A for g^{t+1} runs.
 * ihs_ols_factor: Hinv = (scale^2 SA^T SA)^{-1}, d x d row-major (full,
 * symmetric), through the Cholesky factor (Hinv = L^{-T} L^{-1}), in one
 * thread-block-cluster launch on the ctx's high-priority factor stream,
 * ordered after all work already enqueued on the ctx stream.  d <= 128 (else
 * IHS_ERR_UNSUPPORTED), m >= 1.  Not positive definite: IHS_ERR_NOT_SPD
 * (device status) and Hinv = 0.  SA must stay unmodified, and Hinv unread,
 * until the factor is joined into the ctx stream: by an ihs_ols_apply on the
 * same Hinv, or ihs_ctx_synchronize / ihs_ctx_destroy on this ctx.  Several
 * factors (distinct Hinv) may be in flight.
 * ihs_ols_apply: x_next = x + Hinv g (one CTA; d <= 1024), after the pending
 * factor that writes this Hinv, if any.  x_next may alias x. */
ihs_status ihs_ols_factor(ihs_ctx ctx, const double *SA, int64_t m, int64_t d, double scale,
                          double *Hinv);
ihs_status ihs_ols_apply(ihs_ctx ctx, const double *Hinv, const double *g, int64_t d,
                         const double *x, double *x_next);

/* Look-ahead Gram for the l1-ball / LASSO updates: H = scale^2 SA^T SA (d x d)
 * on the factor stream (as ihs_ols_factor, with a Gram plan for a few SMs so it
 * runs beside other work).  Joined by the next ihs_l1ball_update /
 * ihs_lasso_update / ihs_ols_update / ihs_ols_apply that reads this H, or by
 * ihs_ctx_synchronize / ihs_ctx_destroy. */
ihs_status ihs_gram_lookahead(ihs_ctx ctx, const double *SA, int64_t m, int64_t d, double scale,
                              double *H);

/* One look-ahead OLS step on one rank (nothing to all-reduce): the pass over A
 * (dense) at x forms g = A^T (b - A x) (written to g, d) and, if SA_next is
 * not NULL, S^{iter_next} A into SA_next (m x d, as ihs_sketch); if Hinv_next
 * is also not NULL, ihs_ols_factor(SA_next -> Hinv_next) is enqueued as soon
 * as SA_next is complete; then x_next = x + Hinv g, where Hinv is the factor
 * of the current iteration's sketch (its pending factor is joined first).  The
 * gradient reduction and the update are one launch.  Iterating
 *   x^{t+1} = step(iter_next = t + 1, x^t, Hinv = H_t^{-1}, -> H_{t+1}^{-1})
 * after a prologue ihs_sketch(t0) + ihs_ols_factor gives the IHS iterates of
 * ihs_solve_ols.  Statuses as for ihs_ols_factor / ihs_sketch_grad. */
ihs_status ihs_ols_lookahead_step(ihs_ctx ctx, const ihs_matrix *A, const ihs_sketch_spec *spec,
                                  uint64_t iter_next, const double *b, const double *x,
                                  const double *Hinv, double *SA_next, double *Hinv_next,
                                  double *g, double *x_next);

/* a1-a6 of one OLS iteration of a small dense problem in ONE launch of one CTA
 * (small_step.cu; the path of ihs_solve_ols for such problems, option
 * "small_step"): SA = S^(iter) A (s blocks, 1/sqrt(s)), g = A^T (b - A x),
 * H = SA^T SA, x_next = x + H^{-1} g (Cholesky).  d <= 32, n <= 32768 and the
 * working set within one CTA's shared memory, else IHS_ERR_UNSUPPORTED.
 * SA_out (m x d), g_out (d), H_out (d x d) may be NULL.  One rank (the local
 * rows only: no all-reduce).  Statuses as for ihs_ols_update. */
ihs_status ihs_small_step(ihs_ctx ctx, const ihs_matrix *A, const double *b, const ihs_sketch_spec *spec,
                          uint64_t iter, const double *x, double *x_next, double *SA_out, double *g_out,
                          double *H_out);

/* a6, OLS: x_next = x + H^{-1} g (Eq. (2) with C = R^d; the
 * QP "solved exactly").  d <= 160: blocked Cholesky in one
 * CTA; d > 160: one cooperative launch per the "ols_large" option (default:
 * Jacobi-preconditioned CG to a relative residual of 1e-15, falling back to
 * the blocked Cholesky in the same launch when CG hits its cap min(2000, 4d)
 * or meets p.Hp <= 0; reading R22).  H not positive definite (a Cholesky pivot
 * <= 0) sets IHS_ERR_NOT_SPD (device status) and writes x_next = x (reading
 * R13).  H is not modified.  x_next may alias x. */
ihs_status ihs_ols_update(ihs_ctx ctx, const double *H, const double *g, int64_t d,
                          const double *x, double *x_next);

/* a6, l1 ball {||x||_1 <= radius}: projected gradient on
 * 1/2 (y-x)^T H (y-x) - g^T (y-x) (reading R10).  inner_iters (device int32,
 * may be NULL) receives the step count; the cap sets IHS_ERR_NOT_CONVERGED
 * (device status) with the last iterate written. */
ihs_status ihs_l1ball_update(ihs_ctx ctx, const double *H, const double *g, int64_t d,
                             const double *x, double radius, const ihs_inner_cfg *cfg,
                             double *x_next, int32_t *inner_iters);

/* NEXT-2, penalised LASSO (section 3: 1/2||Ax-b||^2 +
 * lambda ||x||_1; the penalty is carried into every IHS step, reading R23):
 * x_next = argmin_y 1/2 (y-x)^T H (y-x) - g^T (y-x) + lambda ||y||_1 by
 * accelerated proximal gradient (soft threshold at lambda / L; L, start,
 * stopping rule and cap as for the ball, reading R10).  lambda >= 0;
 * d <= 256 (else IHS_ERR_UNSUPPORTED).  inner_iters / statuses as for
 * ihs_l1ball_update. */
ihs_status ihs_lasso_update(ihs_ctx ctx, const double *H, const double *g, int64_t d,
                            const double *x, double lambda, const ihs_inner_cfg *cfg,
                            double *x_next, int32_t *inner_iters);

/* a1-a7, Iterative Hessian Sketch (Eq. (2), section 1; a fresh
 * sketch S^{t+1} per iteration, the exact gradient A^T(b - A x^t)):
 * x^{t+1} = argmin_{x in C} 1/2 ||S^{t+1} A (x - x^t)||^2 - <A^T(b - A x^t), x - x^t>,
 * n_iters steps from x0 (NULL = 0, reading R11), hash iterations iter0.. .
 * ihs_solve_ols: C = R^d (the ihs_ols_update step).
 * A/b/x0/x/x_hist may be HOST or DEVICE pointers (detected per pointer); host
 * inputs are copied in and results copied out inside the call.  x_hist
 * (optional, (n_iters+1) x d) receives x^0..x^T.  trace (host, optional)
 * receives n_iters records and makes the call synchronous (plain schedule).
 * With a communicator set, [SA | g] is summed across ranks every iteration and
 * every rank computes the same x; the schedule (plain or look-ahead, option
 * "lookahead") is decided from ceil(n_global / world) rows so that all ranks
 * take the same one.  Returns after the last step is enqueued (or completed
 * when any host pointer or trace is involved).  Errors: argument errors
 * synchronously; IHS_ERR_NOT_SPD / IHS_ERR_NOT_CONVERGED of the inner steps at
 * the next ihs_ctx_synchronize (or returned, when the call is synchronous). */
ihs_status ihs_solve_ols(ihs_ctx ctx, const ihs_matrix *A, const double *b,
                         const ihs_sketch_spec *spec, int32_t n_iters, uint64_t iter0,
                         const double *x0, double *x, double *x_hist,
                         ihs_iter_record *trace);

/* The same loop with C = {||x||_1 <= radius} (the LASSO constraint of the
 * paper's Eq. (1) setting; BASELINE.json configs[3]), each QP
 * solved by ihs_l1ball_update with cfg (NULL = defaults). */
ihs_status ihs_solve_l1ball(ihs_ctx ctx, const ihs_matrix *A, const double *b, double radius,
                            const ihs_sketch_spec *spec, int32_t n_iters, uint64_t iter0,
                            const ihs_inner_cfg *cfg, const double *x0, double *x,
                            double *x_hist, ihs_iter_record *trace);

/* NEXT-2: the same loop for the penalised LASSO 1/2||Ax - b||^2 + lambda ||x||_1
 * (section 3; the penalty kept in every step, reading R23),
 * each QP solved by ihs_lasso_update. */
ihs_status ihs_solve_lasso(ihs_ctx ctx, const ihs_matrix *A, const double *b, double lambda,
                           const ihs_sketch_spec *spec, int32_t n_iters, uint64_t iter0,
                           const ihs_inner_cfg *cfg, const double *x0, double *x,
                           double *x_hist, ihs_iter_record *trace);

/* a7 bookkeeping: err2[k] = ||A_local (X[k] - xref)||^2 and ref2 = ||A_local xref||^2
 * for k < count (X is count x d, device).  One pass over A.  Summed across
 * ranks by the caller; e_k = sqrt(err2[k] / ref2). */
ihs_status ihs_pred_err2(ihs_ctx ctx, const ihs_matrix *A, const double *X, int32_t count,
                         const double *xref, double *err2, double *ref2);

#ifdef __cplusplus
}
#endif
#endif /* IHS_H */
