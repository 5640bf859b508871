/*
 * oracle/ihs_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, sequential, fp64 CPU oracle for the Iterative Hessian Sketch
 * (IHS) hot path of arXiv 1910.14166 ("Iterative Hessian Sketch with sparse
 * embeddings"; /root/reference/PAPER.md).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load or execute this
 * library.  It shares no source, header, table or helper with the CUDA product
 * path (paper_1910_14166_b200/csrc) and neither imports the other.
 *
 * Every loop runs in the order the paper / DESIGN.md readings state, with no
 * blocking, fusion or reordering.  Compiled with -O2 -ffp-contract=off so each
 * a*b+c is two roundings, exactly as written.
 *
 * Citations are PAPER.md line numbers with the section they fall in; "R<k>" are
 * the readings listed in DESIGN.md section 3 (the paper is silent or garbled there).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_ERR_INVALID 1
#define OR_ERR_NOT_SPD 3
#define OR_ERR_NOT_CONVERGED 4

/* ------------------------------------------------------------------------ */
/* Counter hash (R1: BASELINE.json north_star "splitmix64 of seed, iteration,
 * global row index"; the paper itself draws h(i), sigma(i) "uniformly at
 * random", section 2).                                      */
/* ------------------------------------------------------------------------ */

/* splitmix64 step: add the golden gamma, then the finaliser. */
uint64_t or_splitmix64(uint64_t x)
{
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* Per-iteration key k_t = SM(SM(seed) xor t)   (R1, R2: t = 0 for x^0 -> x^1). */
uint64_t or_iter_key(uint64_t seed, uint64_t t)
{
    return or_splitmix64(or_splitmix64(seed) ^ t);
}

/* Bucket and sign of global row i in SJLT block j (CountSketch is s = 1).
 * SJLT = s stacked independent CountSketches of m/s rows;
 * block j owns rows [j*m/s, (j+1)*m/s).  w = SM(k_t xor (i*s + j));
 * bucket = j*M + floor(hi32(w) * M / 2^32); sign = +1 iff bit 0 of w is 0.  */
void or_hash(uint64_t key, int64_t i, int32_t j, int32_t s, int64_t m,
             int64_t *bucket, int32_t *sign)
{
    uint64_t w = or_splitmix64(key ^ ((uint64_t)i * (uint64_t)s + (uint64_t)j));
    uint64_t M = (uint64_t)(m / s);
    *bucket = (int64_t)j * (int64_t)M + (int64_t)(((w >> 32) * M) >> 32);
    *sign = (w & 1ULL) ? -1 : 1;
}

/* Export the hash for rows [row_begin, row_begin+count): arrays of count*s,
 * row-major (row, block). */
void or_hash_rows(uint64_t seed, uint64_t t, int32_t s, int64_t m,
                  int64_t row_begin, int64_t count, int32_t *bucket, int8_t *sign)
{
    uint64_t key = or_iter_key(seed, t);
    for (int64_t r = 0; r < count; ++r) {
        for (int32_t j = 0; j < s; ++j) {
            int64_t b; int32_t sg;
            or_hash(key, row_begin + r, j, s, m, &b, &sg);
            bucket[r * s + j] = (int32_t)b;
            sign[r * s + j] = (int8_t)sg;
        }
    }
}

/* ------------------------------------------------------------------------ */
/* a2: the sketch SA = S A (section 2 definitions; streaming
 * application "bucket h(i) accumulates +-row i", PAPER.md:236-240 read per
 * R6; SJLT normalised by 1/sqrt(s), appendix A.1.1, R5).    */
/* ------------------------------------------------------------------------ */

/* Explicit (h, sigma) form: bucket/sign hold n*s entries.  Sum in ascending
 * row order, then scale every finished element by 1/sqrt(s) once. */
void or_sketch_dense_hs(int64_t n, int64_t d, const double *A, int64_t m, int32_t s,
                        const int32_t *bucket, const int8_t *sign, double *SA)
{
    memset(SA, 0, sizeof(double) * (size_t)(m * d));
    for (int64_t i = 0; i < n; ++i)
        for (int32_t j = 0; j < s; ++j) {
            int64_t b = bucket[i * s + j];
            double sg = (double)sign[i * s + j];
            for (int64_t c = 0; c < d; ++c)
                SA[b * d + c] += sg * A[i * d + c];
        }
    if (s > 1) {
        double scale = 1.0 / sqrt((double)s);
        for (int64_t e = 0; e < m * d; ++e) SA[e] = SA[e] * scale;
    }
}

/* Hash-defined sketch of a dense row-major n x d block whose first row has
 * global index row_offset. */
void or_sketch_dense(int64_t n, int64_t d, const double *A, int64_t row_offset,
                     uint64_t seed, uint64_t t, int64_t m, int32_t s, double *SA)
{
    uint64_t key = or_iter_key(seed, t);
    memset(SA, 0, sizeof(double) * (size_t)(m * d));
    for (int64_t i = 0; i < n; ++i)
        for (int32_t j = 0; j < s; ++j) {
            int64_t b; int32_t sg;
            or_hash(key, row_offset + i, j, s, m, &b, &sg);
            for (int64_t c = 0; c < d; ++c)
                SA[b * d + c] += (double)sg * A[i * d + c];
        }
    if (s > 1) {
        double scale = 1.0 / sqrt((double)s);
        for (int64_t e = 0; e < m * d; ++e) SA[e] = SA[e] * scale;
    }
}

/* Only the SA rows listed in `rows` (sampled outputs at full size).  out is
 * nrows x d.  Same per-element order as or_sketch_dense. */
void or_sketch_dense_rows(int64_t n, int64_t d, const double *A, int64_t row_offset,
                          uint64_t seed, uint64_t t, int64_t m, int32_t s,
                          int64_t nrows, const int64_t *rows, double *out)
{
    uint64_t key = or_iter_key(seed, t);
    memset(out, 0, sizeof(double) * (size_t)(nrows * d));
    for (int64_t i = 0; i < n; ++i)
        for (int32_t j = 0; j < s; ++j) {
            int64_t b; int32_t sg;
            or_hash(key, row_offset + i, j, s, m, &b, &sg);
            for (int64_t q = 0; q < nrows; ++q)
                if (rows[q] == b)
                    for (int64_t c = 0; c < d; ++c)
                        out[q * d + c] += (double)sg * A[i * d + c];
        }
    if (s > 1) {
        double scale = 1.0 / sqrt((double)s);
        for (int64_t e = 0; e < nrows * d; ++e) out[e] = out[e] * scale;
    }
}

/* CSR A: row_ptr[n+1] (row_ptr[0] = 0), col[nnz], val[nnz].  Every stored
 * entry of row i is added into each of its s buckets ("touch each stored
 * nonzero s times"). */
void or_sketch_csr(int64_t n, int64_t d, const int64_t *row_ptr, const int32_t *col,
                   const double *val, int64_t row_offset, uint64_t seed, uint64_t t,
                   int64_t m, int32_t s, double *SA)
{
    uint64_t key = or_iter_key(seed, t);
    memset(SA, 0, sizeof(double) * (size_t)(m * d));
    for (int64_t i = 0; i < n; ++i)
        for (int32_t j = 0; j < s; ++j) {
            int64_t b; int32_t sg;
            or_hash(key, row_offset + i, j, s, m, &b, &sg);
            for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e)
                SA[b * d + col[e]] += (double)sg * val[e];
        }
    if (s > 1) {
        double scale = 1.0 / sqrt((double)s);
        for (int64_t e = 0; e < m * d; ++e) SA[e] = SA[e] * scale;
    }
}

/* ------------------------------------------------------------------------ */
/* a5: g = A^T (b - A x), the linear term of Eq. (2) (section 1;
 * sign convention R21: ihs_grad returns +A^T(b - Ax) = -grad f).            */
/* ------------------------------------------------------------------------ */
void or_grad_dense(int64_t n, int64_t d, const double *A, const double *b,
                   const double *x, double *g)
{
    memset(g, 0, sizeof(double) * (size_t)d);
    for (int64_t i = 0; i < n; ++i) {
        double ax = 0.0;
        for (int64_t c = 0; c < d; ++c) ax += A[i * d + c] * x[c];
        double r = b[i] - ax;
        for (int64_t c = 0; c < d; ++c) g[c] += A[i * d + c] * r;
    }
}

void or_grad_csr(int64_t n, int64_t d, const int64_t *row_ptr, const int32_t *col,
                 const double *val, const double *b, const double *x, double *g)
{
    memset(g, 0, sizeof(double) * (size_t)d);
    for (int64_t i = 0; i < n; ++i) {
        double ax = 0.0;
        for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) ax += val[e] * x[col[e]];
        double r = b[i] - ax;
        for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) g[col[e]] += val[e] * r;
    }
}

/* Residual vector r = b - A x (used by the error norm, a7). */
void or_matvec_dense(int64_t n, int64_t d, const double *A, const double *x, double *y)
{
    for (int64_t i = 0; i < n; ++i) {
        double acc = 0.0;
        for (int64_t c = 0; c < d; ++c) acc += A[i * d + c] * x[c];
        y[i] = acc;
    }
}

void or_matvec_csr(int64_t n, const int64_t *row_ptr, const int32_t *col,
                   const double *val, const double *x, double *y)
{
    for (int64_t i = 0; i < n; ++i) {
        double acc = 0.0;
        for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) acc += val[e] * x[col[e]];
        y[i] = acc;
    }
}

/* ------------------------------------------------------------------------ */
/* a4: the approximate Hessian H = (SA)^T SA (section 1). */
/* ------------------------------------------------------------------------ */
void or_gram(int64_t m, int64_t d, const double *SA, double *H)
{
    for (int64_t p = 0; p < d; ++p)
        for (int64_t q = p; q < d; ++q) {
            double acc = 0.0;
            for (int64_t r = 0; r < m; ++r) acc += SA[r * d + p] * SA[r * d + q];
            H[p * d + q] = acc;
            H[q * d + p] = acc;
        }
}

/* ------------------------------------------------------------------------ */
/* a6 (OLS, C = R^d): x^{t+1} = x^t + H^{-1} g, Eq. (2) with no constraint.  */
/* Textbook column Cholesky H = L L^T; a pivot <= 0 is an error (R13).       */
/* ------------------------------------------------------------------------ */
int or_cholesky(int64_t d, const double *H, double *L)
{
    memset(L, 0, sizeof(double) * (size_t)(d * d));
    for (int64_t j = 0; j < d; ++j) {
        double s = H[j * d + j];
        for (int64_t k = 0; k < j; ++k) s -= L[j * d + k] * L[j * d + k];
        if (!(s > 0.0)) return OR_ERR_NOT_SPD;
        double ljj = sqrt(s);
        L[j * d + j] = ljj;
        for (int64_t i = j + 1; i < d; ++i) {
            double t = H[i * d + j];
            for (int64_t k = 0; k < j; ++k) t -= L[i * d + k] * L[j * d + k];
            L[i * d + j] = t / ljj;
        }
    }
    return OR_OK;
}

/* Solve L L^T u = g: forward L y = g, backward L^T u = y. */
void or_chol_solve(int64_t d, const double *L, const double *g, double *u)
{
    double *y = (double *)malloc(sizeof(double) * (size_t)d);
    for (int64_t i = 0; i < d; ++i) {
        double t = g[i];
        for (int64_t k = 0; k < i; ++k) t -= L[i * d + k] * y[k];
        y[i] = t / L[i * d + i];
    }
    for (int64_t i = d - 1; i >= 0; --i) {
        double t = y[i];
        for (int64_t k = i + 1; k < d; ++k) t -= L[k * d + i] * u[k];
        u[i] = t / L[i * d + i];
    }
    free(y);
}

int or_ols_step(int64_t d, const double *H, const double *g, const double *x, double *x_next)
{
    double *L = (double *)malloc(sizeof(double) * (size_t)(d * d));
    double *u = (double *)malloc(sizeof(double) * (size_t)d);
    int st = or_cholesky(d, H, L);
    if (st == OR_OK) {
        or_chol_solve(d, L, g, u);
        for (int64_t c = 0; c < d; ++c) x_next[c] = x[c] + u[c];
    }
    free(L); free(u);
    return st;
}

/* ------------------------------------------------------------------------ */
/* a6 (l1 ball, C = {||x||_1 <= tau}, section 1).            */
/* ------------------------------------------------------------------------ */

static int or_cmp_desc(const void *a, const void *b)
{
    double x = *(const double *)a, y = *(const double *)b;
    return (x < y) - (x > y);
}

/* Euclidean projection onto {||x||_1 <= tau} by the sorted-threshold rule
 * (R8): sort |v| descending -> u; rho = max{k : u_k > (sum_{r<=k} u_r - tau)/k};
 * theta = (sum_{r<=rho} u_r - tau)/rho; out = sign(v) max(|v| - theta, 0). */
void or_project_l1(int64_t d, const double *v, double tau, double *out)
{
    double norm1 = 0.0;
    for (int64_t c = 0; c < d; ++c) norm1 += fabs(v[c]);
    if (norm1 <= tau) {
        for (int64_t c = 0; c < d; ++c) out[c] = v[c];
        return;
    }
    double *u = (double *)malloc(sizeof(double) * (size_t)d);
    for (int64_t c = 0; c < d; ++c) u[c] = fabs(v[c]);
    qsort(u, (size_t)d, sizeof(double), or_cmp_desc);
    /* k = 1 always satisfies the rule when tau > 0; for tau = 0 the set is empty
     * and theta = u_1 maps the ball {0} correctly (every entry thresholds to 0). */
    double csum = 0.0, theta = u[0] - tau;
    for (int64_t k = 1; k <= d; ++k) {
        csum += u[k - 1];
        double t = (csum - tau) / (double)k;
        if (u[k - 1] > t) theta = t;
    }
    free(u);
    if (theta < 0.0) theta = 0.0;
    for (int64_t c = 0; c < d; ++c) {
        double a = fabs(v[c]) - theta;
        out[c] = a > 0.0 ? (v[c] < 0.0 ? -a : a) : 0.0;
    }
}

/* Largest eigenvalue of symmetric H by power iteration from 1/sqrt(d). */
double or_power_lmax(int64_t d, const double *H, int32_t iters)
{
    double *v = (double *)malloc(sizeof(double) * (size_t)d);
    double *w = (double *)malloc(sizeof(double) * (size_t)d);
    double lam = 0.0;
    for (int64_t c = 0; c < d; ++c) v[c] = 1.0 / sqrt((double)d);
    for (int32_t k = 0; k < iters; ++k) {
        for (int64_t p = 0; p < d; ++p) {
            double acc = 0.0;
            for (int64_t q = 0; q < d; ++q) acc += H[p * d + q] * v[q];
            w[p] = acc;
        }
        double nn = 0.0;
        for (int64_t p = 0; p < d; ++p) nn += w[p] * w[p];
        lam = sqrt(nn);
        if (!(lam > 0.0)) break;
        for (int64_t p = 0; p < d; ++p) v[p] = w[p] / lam;
    }
    free(v); free(w);
    return lam;
}

/* Projected gradient on q(y) = 1/2 (y-x)^T H (y-x) - g^T (y-x) over the ball
 * (R10): L = safety * lambda_max(H); y^0 = x;
 * y^{k+1} = P(y^k - (H(y^k - x) - g)/L) until ||y^{k+1}-y^k||_2 <= tol*max(1,||y^k||_2)
 * or max_inner steps.  Returns OR_ERR_NOT_CONVERGED (with the last iterate)
 * when the cap is hit.  *iters_out = number of steps taken. */
int or_l1ball_step(int64_t d, const double *H, const double *g, const double *x,
                   double tau, int32_t max_inner, double tol, int32_t power_iters,
                   double safety, double *x_next, int32_t *iters_out)
{
    double L = safety * or_power_lmax(d, H, power_iters);
    double *y = (double *)malloc(sizeof(double) * (size_t)d);
    double *z = (double *)malloc(sizeof(double) * (size_t)d);
    double *yn = (double *)malloc(sizeof(double) * (size_t)d);
    int st = OR_ERR_NOT_CONVERGED;
    int32_t k = 0;
    for (int64_t c = 0; c < d; ++c) y[c] = x[c];
    while (k < max_inner) {
        for (int64_t p = 0; p < d; ++p) {
            double acc = 0.0;
            for (int64_t q = 0; q < d; ++q) acc += H[p * d + q] * (y[q] - x[q]);
            double grad = acc - g[p];
            z[p] = y[p] - grad / L;
        }
        or_project_l1(d, z, tau, yn);
        ++k;
        double dn = 0.0, yy = 0.0;
        for (int64_t c = 0; c < d; ++c) {
            double e = yn[c] - y[c];
            dn += e * e;
            yy += y[c] * y[c];
        }
        for (int64_t c = 0; c < d; ++c) y[c] = yn[c];
        if (sqrt(dn) <= tol * fmax(1.0, sqrt(yy))) { st = OR_OK; break; }
    }
    for (int64_t c = 0; c < d; ++c) x_next[c] = y[c];
    if (iters_out) *iters_out = k;
    free(y); free(z); free(yn);
    return st;
}

/* NEXT-2, penalised LASSO (section 3: x_OPT = argmin
 * 1/2||Ax - b||^2 + lambda ||x||_1; the IHS step keeps the penalty, reading
 * R23): proximal gradient on q(y) + lambda ||y||_1, q as in or_l1ball_step,
 * with the l1 prox (soft-thresholding at lambda / L) in place of the ball
 * projection; same L, start, stopping rule and cap as R10. */
int or_lasso_step(int64_t d, const double *H, const double *g, const double *x,
                  double lambda, int32_t max_inner, double tol, int32_t power_iters,
                  double safety, double *x_next, int32_t *iters_out)
{
    double L = safety * or_power_lmax(d, H, power_iters);
    double *y = (double *)malloc(sizeof(double) * (size_t)d);
    double *yn = (double *)malloc(sizeof(double) * (size_t)d);
    int st = OR_ERR_NOT_CONVERGED;
    int32_t k = 0;
    for (int64_t c = 0; c < d; ++c) y[c] = x[c];
    while (k < max_inner) {
        for (int64_t p = 0; p < d; ++p) {
            double acc = 0.0;
            for (int64_t q = 0; q < d; ++q) acc += H[p * d + q] * (y[q] - x[q]);
            double z = y[p] - (acc - g[p]) / L;
            double a = fabs(z) - lambda / L;                  /* soft threshold */
            yn[p] = a > 0.0 ? (z < 0.0 ? -a : a) : 0.0;
        }
        ++k;
        double dn = 0.0, yy = 0.0;
        for (int64_t c = 0; c < d; ++c) {
            double e = yn[c] - y[c];
            dn += e * e;
            yy += y[c] * y[c];
        }
        for (int64_t c = 0; c < d; ++c) y[c] = yn[c];
        if (sqrt(dn) <= tol * fmax(1.0, sqrt(yy))) { st = OR_OK; break; }
    }
    for (int64_t c = 0; c < d; ++c) x_next[c] = y[c];
    if (iters_out) *iters_out = k;
    free(y); free(yn);
    return st;
}

/* ------------------------------------------------------------------------ */
/* a1-a7 loop (Eq. (2); x^0 = 0 unless given, R11).         */
/* layout: 0 = dense (A = values, n x d), 1 = CSR.  constraint: 0 = OLS,     */
/* 1 = l1 ball of radius tau, 2 = l1 penalty lambda = tau (NEXT-2).          */
/* x_hist is (T+1) x d and receives x^0..x^T.                                 */
/* inner_iters (optional, T entries) receives the PG step counts.             */
/* ------------------------------------------------------------------------ */
int or_ihs_solve(int32_t layout, int64_t n, int64_t d, const double *values,
                 const int64_t *row_ptr, const int32_t *col, const double *b,
                 uint64_t seed, int64_t m, int32_t s, int32_t T, uint64_t iter0,
                 int32_t constraint, double tau, int32_t max_inner, double tol,
                 int32_t power_iters, double safety, const double *x0,
                 double *x_hist, int32_t *inner_iters)
{
    double *SA = (double *)malloc(sizeof(double) * (size_t)(m * d));
    double *H = (double *)malloc(sizeof(double) * (size_t)(d * d));
    double *g = (double *)malloc(sizeof(double) * (size_t)d);
    int st = OR_OK;
    for (int64_t c = 0; c < d; ++c) x_hist[c] = x0 ? x0[c] : 0.0;
    for (int32_t t = 0; t < T; ++t) {
        const double *x = x_hist + (size_t)t * d;
        double *xn = x_hist + (size_t)(t + 1) * d;
        if (layout == 0) {
            or_sketch_dense(n, d, values, 0, seed, iter0 + (uint64_t)t, m, s, SA);
            or_grad_dense(n, d, values, b, x, g);
        } else {
            or_sketch_csr(n, d, row_ptr, col, values, 0, seed, iter0 + (uint64_t)t, m, s, SA);
            or_grad_csr(n, d, row_ptr, col, values, b, x, g);
        }
        or_gram(m, d, SA, H);
        if (constraint == 0) {
            st = or_ols_step(d, H, g, x, xn);
        } else {
            int32_t it = 0;
            if (constraint == 1)
                st = or_l1ball_step(d, H, g, x, tau, max_inner, tol, power_iters, safety, xn, &it);
            else
                st = or_lasso_step(d, H, g, x, tau, max_inner, tol, power_iters, safety, xn, &it);
            if (inner_iters) inner_iters[t] = it;
            if (st == OR_ERR_NOT_CONVERGED) st = OR_OK; /* best iterate kept */
        }
        if (st != OR_OK) break;
    }
    free(SA); free(H); free(g);
    return st;
}

/* ------------------------------------------------------------------------ */
/* O10: exact x_OPT (Eq. (1)).  G = A^T A, c = A^T b in row  */
/* order; OLS: Cholesky solve + one step of iterative refinement.            */
/* ------------------------------------------------------------------------ */
void or_normal_dense(int64_t n, int64_t d, const double *A, const double *b,
                     double *G, double *c)
{
    memset(G, 0, sizeof(double) * (size_t)(d * d));
    memset(c, 0, sizeof(double) * (size_t)d);
    for (int64_t i = 0; i < n; ++i) {
        const double *a = A + i * d;
        for (int64_t p = 0; p < d; ++p) {
            c[p] += a[p] * b[i];
            for (int64_t q = p; q < d; ++q) G[p * d + q] += a[p] * a[q];
        }
    }
    for (int64_t p = 0; p < d; ++p)
        for (int64_t q = 0; q < p; ++q) G[p * d + q] = G[q * d + p];
}

void or_normal_csr(int64_t n, int64_t d, const int64_t *row_ptr, const int32_t *col,
                   const double *val, const double *b, double *G, double *c)
{
    memset(G, 0, sizeof(double) * (size_t)(d * d));
    memset(c, 0, sizeof(double) * (size_t)d);
    for (int64_t i = 0; i < n; ++i)
        for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
            int64_t p = col[e];
            c[p] += val[e] * b[i];
            for (int64_t f = e; f < row_ptr[i + 1]; ++f) {
                int64_t q = col[f];
                G[p * d + q] += val[e] * val[f];
            }
        }
    for (int64_t p = 0; p < d; ++p)
        for (int64_t q = 0; q < p; ++q) G[p * d + q] = G[q * d + p];
}

/* OLS from precomputed (G, c) plus the data for one refinement step. */
int or_exact_ols(int32_t layout, int64_t n, int64_t d, const double *values,
                 const int64_t *row_ptr, const int32_t *col, const double *b,
                 double *x)
{
    double *G = (double *)malloc(sizeof(double) * (size_t)(d * d));
    double *c = (double *)malloc(sizeof(double) * (size_t)d);
    double *L = (double *)malloc(sizeof(double) * (size_t)(d * d));
    double *u = (double *)malloc(sizeof(double) * (size_t)d);
    if (layout == 0) or_normal_dense(n, d, values, b, G, c);
    else or_normal_csr(n, d, row_ptr, col, values, b, G, c);
    int st = or_cholesky(d, G, L);
    if (st == OR_OK) {
        or_chol_solve(d, L, c, x);
        /* one step of iterative refinement: x += G^{-1} A^T (b - A x) */
        if (layout == 0) or_grad_dense(n, d, values, b, x, c);
        else or_grad_csr(n, d, row_ptr, col, values, b, x, c);
        or_chol_solve(d, L, c, u);
        for (int64_t k = 0; k < d; ++k) x[k] += u[k];
    }
    free(G); free(c); free(L); free(u);
    return st;
}

/* l1 ball: IHS with the exact Hessian (S = I), i.e. repeated PG solves of
 * Eq. (2) with H = A^T A, until the outer step stalls below outer_tol. */
int or_exact_l1ball(int32_t layout, int64_t n, int64_t d, const double *values,
                    const int64_t *row_ptr, const int32_t *col, const double *b,
                    double tau, int32_t outer, int32_t max_inner, double tol,
                    double *x)
{
    double *G = (double *)malloc(sizeof(double) * (size_t)(d * d));
    double *c = (double *)malloc(sizeof(double) * (size_t)d);
    double *g = (double *)malloc(sizeof(double) * (size_t)d);
    double *xn = (double *)malloc(sizeof(double) * (size_t)d);
    if (layout == 0) or_normal_dense(n, d, values, b, G, c);
    else or_normal_csr(n, d, row_ptr, col, values, b, G, c);
    int st = OR_OK;
    for (int64_t k = 0; k < d; ++k) x[k] = 0.0;
    for (int32_t t = 0; t < outer; ++t) {
        if (layout == 0) or_grad_dense(n, d, values, b, x, g);
        else or_grad_csr(n, d, row_ptr, col, values, b, x, g);
        int32_t it = 0;
        st = or_l1ball_step(d, G, g, x, tau, max_inner, tol, 50, 1.05, xn, &it);
        double dn = 0.0, xx = 0.0;
        for (int64_t k = 0; k < d; ++k) {
            dn += (xn[k] - x[k]) * (xn[k] - x[k]);
            xx += xn[k] * xn[k];
            x[k] = xn[k];
        }
        if (sqrt(dn) <= 1e-15 * fmax(1.0, sqrt(xx))) break;
    }
    free(G); free(c); free(g); free(xn);
    return st == OR_ERR_NOT_CONVERGED ? OR_OK : st;
}

/* NEXT-2: x_OPT of the penalised LASSO, IHS with the exact Hessian A^T A. */
int or_exact_lasso(int64_t n, int64_t d, const double *A, const double *b, double lambda,
                   int32_t outer, int32_t max_inner, double tol, double *x)
{
    double *G = (double *)malloc(sizeof(double) * (size_t)(d * d));
    double *c = (double *)malloc(sizeof(double) * (size_t)d);
    double *g = (double *)malloc(sizeof(double) * (size_t)d);
    double *xn = (double *)malloc(sizeof(double) * (size_t)d);
    or_normal_dense(n, d, A, b, G, c);
    int st = OR_OK;
    for (int64_t k = 0; k < d; ++k) x[k] = 0.0;
    for (int32_t t = 0; t < outer; ++t) {
        or_grad_dense(n, d, A, b, x, g);
        int32_t it = 0;
        st = or_lasso_step(d, G, g, x, lambda, max_inner, tol, 50, 1.05, xn, &it);
        double dn = 0.0, xx = 0.0;
        for (int64_t k = 0; k < d; ++k) {
            dn += (xn[k] - x[k]) * (xn[k] - x[k]);
            xx += xn[k] * xn[k];
            x[k] = xn[k];
        }
        if (sqrt(dn) <= 1e-15 * fmax(1.0, sqrt(xx))) break;
    }
    free(G); free(c); free(g); free(xn);
    return st == OR_ERR_NOT_CONVERGED ? OR_OK : st;
}

/* O11 / a7: e = ||A(x - xref)||_2 / ||A xref||_2 (prediction seminorm,
 * PAPER.md:45-47 section 1; Definition 2; the 1/sqrt(n)
 * cancels). */
double or_pred_rel_err(int32_t layout, int64_t n, int64_t d, const double *values,
                       const int64_t *row_ptr, const int32_t *col,
                       const double *x, const double *xref)
{
    double num = 0.0, den = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        double a = 0.0, r = 0.0;
        if (layout == 0) {
            for (int64_t c = 0; c < d; ++c) {
                a += values[i * d + c] * (x[c] - xref[c]);
                r += values[i * d + c] * xref[c];
            }
        } else {
            for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
                a += values[e] * (x[col[e]] - xref[col[e]]);
                r += values[e] * xref[col[e]];
            }
        }
        num += a * a;
        den += r * r;
    }
    return sqrt(num) / sqrt(den);
}
