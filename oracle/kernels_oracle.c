/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for parity checks.
 *
 * Plain-C restatement of the reference's five kernel-module contracts
 * (rsvdkit/_kernels.pyx, bound at import by rsvdkit/backend.py:39-43).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library; the product path never does.
 *
 * Build flags mirror the reference's (pkg/setup.py:15-19): -ffp-contract=off
 * -fno-builtin-sin -fno-builtin-cos, so the Gaussian stream is bit-identical
 * to the reference's on the same glibc.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* SplitMix64 finaliser — follows _kernels.pyx:22-28. */
static inline uint64_t splitmix_final(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* Box-Muller Gaussian fill — follows _kernels.pyx:31-53.
 * Writes `count` normals, returns the advanced state. A trailing odd
 * element discards the sine half of its pair. */
uint64_t oracle_gauss_fill(int64_t count, uint64_t state, double *out) {
    const uint64_t golden = 0x9E3779B97F4A7C15ULL;
    const double two_neg53 = 1.0 / 9007199254740992.0;
    const double two_pi = 6.283185307179586;
    int64_t i = 0;
    while (i < count) {
        state += golden;
        uint64_t a = splitmix_final(state);
        state += golden;
        uint64_t b = splitmix_final(state);
        double u1 = (double)((a >> 11) + 1) * two_neg53;
        double u2 = (double)((b >> 11) + 1) * two_neg53;
        double rad = sqrt(-2.0 * log(u1));
        double ang = two_pi * u2;
        out[i++] = rad * cos(ang);
        if (i < count) out[i++] = rad * sin(ang);
    }
    return state;
}

/* Dense row-major product, i-l-j order with a zeroed output —
 * follows _kernels.pyx:56-71. */
void oracle_mm(int64_t m, int64_t kk, int64_t n, const double *a,
               const double *b, double *c) {
    memset(c, 0, sizeof(double) * (size_t)(m * n));
    for (int64_t i = 0; i < m; ++i)
        for (int64_t l = 0; l < kk; ++l) {
            double av = a[i * kk + l];
            const double *brow = b + l * n;
            double *crow = c + i * n;
            for (int64_t j = 0; j < n; ++j) crow[j] += av * brow[j];
        }
}

/* CSR times dense, storage-order accumulation — _kernels.pyx:74-92.
 * Rows are independent, so they are split over OpenMP threads: every output
 * element is summed in the reference's order (bitwise identical to the
 * serial loop). */
void oracle_spmm_nt(int64_t nrows, int64_t m, const int64_t *indptr,
                    const int64_t *col, const double *val, const double *b,
                    double *out) {
    memset(out, 0, sizeof(double) * (size_t)(nrows * m));
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t i = 0; i < nrows; ++i)
        for (int64_t e = indptr[i]; e < indptr[i + 1]; ++e) {
            double v = val[e];
            const double *brow = b + col[e] * m;
            double *orow = out + i * m;
            for (int64_t j = 0; j < m; ++j) orow[j] += v * brow[j];
        }
}

/* CSR-transpose times dense, row-order scatter — _kernels.pyx:95-113.
 * Each OpenMP thread owns a slice of the m output columns and runs the
 * reference's full (i, e) scatter over it, so every output element still
 * accumulates its terms in row order (bitwise identical to the serial loop). */
void oracle_spmm_t(int64_t nrows, int64_t ncols, int64_t m,
                   const int64_t *indptr, const int64_t *col,
                   const double *val, const double *b, double *out) {
    memset(out, 0, sizeof(double) * (size_t)(ncols * m));
#pragma omp parallel
    {
        int64_t nt = 1, t = 0;
#ifdef _OPENMP
        nt = omp_get_num_threads();
        t = omp_get_thread_num();
#endif
        int64_t j0 = m * t / nt, j1 = m * (t + 1) / nt;
        if (j1 > j0)
            for (int64_t i = 0; i < nrows; ++i)
                for (int64_t e = indptr[i]; e < indptr[i + 1]; ++e) {
                    double v = val[e];
                    const double *brow = b + i * m;
                    double *orow = out + col[e] * m;
                    for (int64_t j = j0; j < j1; ++j) orow[j] += v * brow[j];
                }
    }
}

static double offdiag_mass(int64_t n, const double *a) {
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j < n; ++j)
            if (i != j) acc += a[i * n + j] * a[i * n + j];
    return sqrt(acc);
}

/* Cyclic-by-row two-sided Jacobi, in place on symmetric `a`, rotations
 * accumulated into `v` — follows _kernels.pyx:116-192 (stop rule, skip
 * threshold tol*||A||_F*1e-3/n, diagonal update app - t*apq).
 * Returns 1 when converged; *off_out / *sweeps_out as in the reference. */
int oracle_jacobi_sweeps(int64_t n, double *a, double *v, double tol,
                         int max_sweeps, double *off_out, int *sweeps_out) {
    double fro = 0.0;
    for (int64_t i = 0; i < n * n; ++i) fro += a[i] * a[i];
    fro = sqrt(fro);
    double threshold = tol * fro;
    double off = offdiag_mass(n, a);
    *sweeps_out = 0;
    *off_out = off;
    if (n < 2 || off <= threshold) return 1;
    double skip = threshold * 1e-3 / (double)n;
    int sweeps = 0;
    while (sweeps < max_sweeps) {
        for (int64_t p = 0; p < n - 1; ++p)
            for (int64_t q = p + 1; q < n; ++q) {
                double apq = a[p * n + q];
                if (fabs(apq) <= skip) continue;
                double app = a[p * n + p], aqq = a[q * n + q];
                double tau = (aqq - app) / (2.0 * apq);
                double t = tau >= 0.0 ? 1.0 / (tau + sqrt(1.0 + tau * tau))
                                      : -1.0 / (-tau + sqrt(1.0 + tau * tau));
                double c = 1.0 / sqrt(1.0 + t * t);
                double s = t * c;
                for (int64_t r = 0; r < n; ++r) {
                    double x = a[r * n + p], y = a[r * n + q];
                    a[r * n + p] = c * x - s * y;
                    a[r * n + q] = s * x + c * y;
                }
                for (int64_t r = 0; r < n; ++r) {
                    double x = a[p * n + r], y = a[q * n + r];
                    a[p * n + r] = c * x - s * y;
                    a[q * n + r] = s * x + c * y;
                }
                a[p * n + q] = 0.0;
                a[q * n + p] = 0.0;
                a[p * n + p] = app - t * apq;
                a[q * n + q] = aqq + t * apq;
                for (int64_t r = 0; r < n; ++r) {
                    double x = v[r * n + p], y = v[r * n + q];
                    v[r * n + p] = c * x - s * y;
                    v[r * n + q] = s * x + c * y;
                }
            }
        ++sweeps;
        off = offdiag_mass(n, a);
        if (off <= threshold) {
            *off_out = off;
            *sweeps_out = sweeps;
            return 1;
        }
    }
    *off_out = off;
    *sweeps_out = sweeps;
    return 0;
}
