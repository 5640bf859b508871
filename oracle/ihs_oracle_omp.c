/*
 * oracle/ihs_oracle_omp.c -- TEST / BASELINE INFRASTRUCTURE ONLY (see
 * oracle/__init__.py).  OpenMP timing variants of the two row-parallel phases
 * of the oracle ("with OpenMP on all host cores, for the
 * row-parallel phases only"), for bench.py's cpu_baseline leg:
 *   or_sketch_dense_omp  -- S A (1/sqrt(s))
 *   or_grad_dense_omp    -- A^T (b - A x) (Eq. (2) linear term)
 * Thread k of T takes the contiguous rows [k n / T, (k+1) n / T), sums into its
 * own partial exactly as or_sketch_dense / or_grad_dense do, and the partials
 * are added in thread order (a fixed order for a fixed T; equal to the serial
 * result up to rounding -- tests/test_oracle_sketch.py checks it).
 * The hash is written out again (reading R1) rather than shared with
 * ihs_oracle.c so the file stands alone; tests pin it to the serial oracle.
 */
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static uint64_t sm64(uint64_t x)
{
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

int or_omp_threads(void) { return omp_get_max_threads(); }

void or_sketch_dense_omp(int64_t n, int64_t d, const double *A, int64_t row_offset,
                         uint64_t seed, uint64_t t, int64_t m, int32_t s, double *SA)
{
    const uint64_t key = sm64(sm64(seed) ^ t);
    const int64_t M = m / s;
    const int T = omp_get_max_threads();
    double *part = (double *)calloc((size_t)T * (size_t)(m * d), sizeof(double));
#pragma omp parallel num_threads(T)
    {
        const int k = omp_get_thread_num();
        double *P = part + (size_t)k * (size_t)(m * d);
        const int64_t i0 = n * k / T, i1 = n * (k + 1) / T;
        for (int64_t i = i0; i < i1; ++i)
            for (int32_t j = 0; j < s; ++j) {
                const uint64_t w = sm64(key ^ ((uint64_t)(row_offset + i) * (uint64_t)s + (uint64_t)j));
                const int64_t b = j * M + (int64_t)(((w >> 32) * (uint64_t)M) >> 32);
                const double sg = (w & 1ull) ? -1.0 : 1.0;
                for (int64_t c = 0; c < d; ++c) P[b * d + c] += sg * A[i * d + c];
            }
    }
    memset(SA, 0, sizeof(double) * (size_t)(m * d));
    for (int k = 0; k < T; ++k)
        for (int64_t e = 0; e < m * d; ++e) SA[e] += part[(size_t)k * (size_t)(m * d) + e];
    if (s > 1) {
        const double scale = 1.0 / sqrt((double)s);
        for (int64_t e = 0; e < m * d; ++e) SA[e] = SA[e] * scale;
    }
    free(part);
}

void or_grad_dense_omp(int64_t n, int64_t d, const double *A, const double *b, const double *x, double *g)
{
    const int T = omp_get_max_threads();
    double *part = (double *)calloc((size_t)T * (size_t)d, sizeof(double));
#pragma omp parallel num_threads(T)
    {
        const int k = omp_get_thread_num();
        double *P = part + (size_t)k * (size_t)d;
        const int64_t i0 = n * k / T, i1 = n * (k + 1) / T;
        for (int64_t i = i0; i < i1; ++i) {
            double ax = 0.0;
            for (int64_t c = 0; c < d; ++c) ax += A[i * d + c] * x[c];
            const double r = b[i] - ax;
            for (int64_t c = 0; c < d; ++c) P[c] += A[i * d + c] * r;
        }
    }
    memset(g, 0, sizeof(double) * (size_t)d);
    for (int k = 0; k < T; ++k)
        for (int64_t c = 0; c < d; ++c) g[c] += part[(size_t)k * (size_t)d + c];
    free(part);
}
