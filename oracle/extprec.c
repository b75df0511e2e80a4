/* TEST INFRASTRUCTURE ONLY — extended-precision oracles (the
 * reference's tests pin its numerics with MPFR-based `exact_dot` /
 * `exact_dot_ratio` / `HighPrecCg` (proj/tests/oracles.hpp), which cannot be
 * built here — no MPFR/GMP; this restates them with gcc's __float128).
 *
 * A product of two doubles is exact in binary128 (106 of 113 significand
 * bits), so a binary128 accumulation of n products carries a relative error
 * of ~n * 2^-113: rounded once to double it is the exactly rounded value
 * except under catastrophic cancellation, which the tests avoid.
 */
#include <stdint.h>
#include <stdlib.h>

typedef __float128 q;

/* <x, y>, exactly rounded (proj/tests/oracles.hpp exact_dot) */
double xp_dot(int64_t n, const double* x, const double* y) {
    q s = 0;
    for (int64_t i = 0; i < n; ++i) s += (q)x[i] * (q)y[i];
    return (double)s;
}

/* sum |x_i y_i| (the scale of the rounding-error bounds) */
double xp_abs_dot(int64_t n, const double* x, const double* y) {
    q s = 0;
    for (int64_t i = 0; i < n; ++i) {
        q t = (q)x[i] * (q)y[i];
        s += t < 0 ? -t : t;
    }
    return (double)s;
}

/* <a, b> / <c, d> in binary128, rounded once (oracles.hpp exact_dot_ratio) */
double xp_ratio(int64_t n, const double* a, const double* b, const double* c, const double* d) {
    q num = 0, den = 0;
    for (int64_t i = 0; i < n; ++i) {
        num += (q)a[i] * (q)b[i];
        den += (q)c[i] * (q)d[i];
    }
    return (double)(num / den);
}

/* Preconditioned CG (paper Alg. 1, the HS recurrences) carried entirely in
 * binary128 on the double-precision A, b, x0 and M = diag(inv_diag) (NULL:
 * identity) — oracles.hpp HighPrecCg. Writes x_k for k = 1..steps (row-major
 * [steps][n]) into xs; returns the number of steps taken (stops early on an
 * exact zero residual or a non-positive curvature). */
int xp_cg(int64_t n, const int64_t* rp, const int64_t* ci, const double* va, const double* inv_diag,
          const double* b, const double* x0, int steps, double* xs) {
    q* x = malloc(sizeof(q) * n);
    q* r = malloc(sizeof(q) * n);
    q* z = malloc(sizeof(q) * n);
    q* p = malloc(sizeof(q) * n);
    q* s = malloc(sizeof(q) * n);
    int k = 0;
    if (!x || !r || !z || !p || !s) goto done;
    for (int64_t i = 0; i < n; ++i) x[i] = x0[i];
    for (int64_t i = 0; i < n; ++i) {
        q t = 0;
        for (int64_t e = rp[i]; e < rp[i + 1]; ++e) t += (q)va[e] * x[ci[e]];
        r[i] = (q)b[i] - t;
        z[i] = inv_diag ? (q)inv_diag[i] * r[i] : r[i];
        p[i] = z[i];
    }
    q nu = 0;
    for (int64_t i = 0; i < n; ++i) nu += z[i] * r[i];
    for (k = 0; k < steps; ++k) {
        if (nu <= 0) break;
        q mu = 0;
        for (int64_t i = 0; i < n; ++i) {
            q t = 0;
            for (int64_t e = rp[i]; e < rp[i + 1]; ++e) t += (q)va[e] * p[ci[e]];
            s[i] = t;
            mu += p[i] * t;
        }
        if (mu <= 0) break;
        const q alpha = nu / mu;
        q nu1 = 0;
        for (int64_t i = 0; i < n; ++i) {
            x[i] += alpha * p[i];
            r[i] -= alpha * s[i];
            z[i] = inv_diag ? (q)inv_diag[i] * r[i] : r[i];
            nu1 += z[i] * r[i];
        }
        const q beta = nu1 / nu;
        nu = nu1;
        for (int64_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
        for (int64_t i = 0; i < n; ++i) xs[(int64_t)k * n + i] = (double)x[i];
    }
done:
    free(x);
    free(r);
    free(z);
    free(p);
    free(s);
    return k;
}
