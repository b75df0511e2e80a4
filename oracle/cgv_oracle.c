/* TEST INFRASTRUCTURE ONLY — CPU oracle for the PCG-variant hot path.
 * See cgv_oracle.h. Every function cites the reference lines it restates
 * (paths relative to /root/reference/proj). Compiled with -ffp-contract=off:
 * every a*x+y below is a rounded multiply followed by a rounded add, as in the
 * reference build (CMakeLists.txt:12-14). */
#define _POSIX_C_SOURCE 199309L
#include "cgv_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* enum values follow inc/variants.hpp:17-86 */
enum { V_HS, V_CG_CG, V_M, V_PR, V_GV, V_PIPE_PR_M, V_PIPE_PR };
enum { NU_EXPANDED, NU_SIMPLIFIED, NU_MEURANT };
enum { ST_RUNNING, ST_BREAKDOWN, ST_MAXITER, ST_CONVERGED };
enum { BR_NONE, BR_NUPRIME, BR_NU, BR_MU, BR_NONFINITE };
enum { CB_ZERO, CB_ERROR, CB_STAGNATION };

/* ---------------------------------------------------------------- dots */

/* vector_ops.hpp:20-25 — left-to-right accumulation */
static double dot_seq(int64_t n, const double* x, const double* y) {
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) acc += x[i] * y[i];
    return acc;
}

/* One CTA's tree over `block` per-thread values: shfl_down 16,8,4,2,1 inside
 * each warp, then warp 0 folds the nw warp sums with offsets nw/2..1. */
static double block_tree(double* v, int block) {
    const int nw = block / 32;
    double wsum[32];
    for (int w = 0; w < nw; ++w) {
        double* a = v + 32 * w;
        for (int off = 16; off >= 1; off >>= 1)
            for (int l = 0; l < off; ++l) a[l] = a[l] + a[l + off];
        wsum[w] = a[0];
    }
    for (int off = nw / 2; off >= 1; off >>= 1)
        for (int l = 0; l < off; ++l) wsum[l] = wsum[l] + wsum[l + off];
    return wsum[0];
}

static double dot_tree(int64_t n, const double* x, const double* y, int block, int gmax,
                       int order) {
    const int64_t ntiles = (n + block - 1) / block;
    if (ntiles == 0) return 0.0;
    const int64_t G = ntiles < gmax ? ntiles : gmax;
    double* partial = (double*)malloc(sizeof(double) * (size_t)G);
    double* v = (double*)malloc(sizeof(double) * (size_t)block);
    for (int64_t b = 0; b < G; ++b) {
        /* thread t of CTA b: sequential sum over rows tile*block+t of its
         * tiles — b, b+G, b+2G, ... (order 0) or the contiguous block
         * [b*ntiles/G, (b+1)*ntiles/G) (order 1); rows >= n add nothing */
        const int64_t lo = order ? b * ntiles / G : b;
        const int64_t hi = order ? (b + 1) * ntiles / G : ntiles;
        const int64_t step = order ? 1 : G;
        for (int t = 0; t < block; ++t) {
            double acc = 0.0;
            for (int64_t tile = lo; tile < hi; tile += step) {
                const int64_t row = tile * block + t;
                if (row < n) acc = acc + x[row] * y[row];
            }
            v[t] = acc;
        }
        partial[b] = block_tree(v, block);
    }
    for (int t = 0; t < block; ++t) {
        double f = 0.0;
        for (int64_t j = t; j < G; j += block) f = f + partial[j];
        v[t] = f;
    }
    const double out = block_tree(v, block);
    free(v);
    free(partial);
    return out;
}

double orc_dot(int64_t n, const double* x, const double* y, const orc_dotcfg* cfg) {
    if (!cfg || cfg->mode == ORC_DOT_SEQ) return dot_seq(n, x, y);
    if (cfg->mode == ORC_DOT_TREE) return dot_tree(n, x, y, cfg->block, cfg->gmax, cfg->order);
    double acc = 0.0; /* rank-ordered sum of per-block trees */
    for (int p = 0; p < cfg->nparts; ++p) {
        const int64_t lo = cfg->part_lo[p], hi = cfg->part_lo[p + 1];
        acc = acc + dot_tree(hi - lo, x + lo, y + lo, cfg->block, cfg->gmax, cfg->order);
    }
    return acc;
}

/* ------------------------------------------------------- L1 primitives */

/* sparse_matrix.cpp:109-118 — per-row left-to-right sum, no contraction */
void orc_spmv(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
              const double* x, double* y) {
    for (int64_t i = 0; i < n; ++i) {
        double sum = 0.0;
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k) sum += v[k] * x[ci[k]];
        y[i] = sum;
    }
}

/* sparse_matrix.cpp:126-143 — one traversal, each output equal to spmv */
void orc_block_spmv(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                    const double* x1, const double* x2, double* y1, double* y2) {
    for (int64_t i = 0; i < n; ++i) {
        double s1 = 0.0, s2 = 0.0;
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
            s1 += v[k] * x1[ci[k]];
            s2 += v[k] * x2[ci[k]];
        }
        y1[i] = s1;
        y2[i] = s2;
    }
}

/* preconditioner.cpp:12-31 */
int orc_jacobi(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
               double* inv_diag) {
    for (int64_t i = 0; i < n; ++i) {
        int found = 0;
        double d = 0.0;
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k)
            if (ci[k] == i) {
                d = v[k];
                found = 1;
                break;
            }
        if (!found || !(d > 0.0)) return -1;
        inv_diag[i] = 1.0 / d;
    }
    return 0;
}

/* sparse_matrix.cpp:64-82 */
int orc_validate_csr(int64_t n, const int64_t* rp, const int64_t* ci, int64_t nnz) {
    if (n < 0 || rp[0] != 0 || rp[n] != nnz) return -1;
    for (int64_t i = 0; i < n; ++i) {
        if (rp[i] > rp[i + 1]) return -1;
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
            if (ci[k] < 0 || ci[k] >= n) return -1;
            if (k > rp[i] && ci[k] <= ci[k - 1]) return -1;
        }
    }
    return 0;
}

/* -------------------------------------------------------------- solver */

struct orc_solver {
    int64_t n;
    const int64_t *rp, *ci;
    const double* va;
    int variant, nu_expr, recompute_nu, recompute_w, unsimplified_mu, track_delta;
    int prec;
    double* inv_diag;
    orc_dotcfg dcfg;
    int64_t part_copy[65];
    int k, state, reason, criterion;
    uint64_t spmv_calls, block_calls, prec_applies, reductions;
    /* x r p s w u t r~ s~ w~ u~ (index = `which` in the C-ABI) */
    double* vec[11];
    double alpha, beta, nu, nu_prime, mu, delta, delta_hat, gamma, eta;
};

enum { X, R, P, S, W, U, T, RT, ST, WT, UT };

static int is_predictor(int v) {
    return v == V_M || v == V_PR || v == V_PIPE_PR_M || v == V_PIPE_PR;
}

/* variants.cpp:35-47 */
int orc_config_validate(int variant, int nu_expr, int recompute_nu, int recompute_w,
                        int unsimplified_mu, int track_delta) {
    const int pipe_pr = variant == V_PIPE_PR || variant == V_PIPE_PR_M;
    if (variant < 0 || variant > V_PIPE_PR) return -1;
    if (!recompute_w && !pipe_pr) return -1;
    if (!recompute_nu && !is_predictor(variant)) return -1;
    if (!is_predictor(variant) && nu_expr != NU_SIMPLIFIED) return -1;
    if (unsimplified_mu && variant != V_CG_CG && variant != V_GV) return -1;
    if (track_delta && !is_predictor(variant)) return -1;
    return 0;
}

/* tilde aliasing of variants.hpp:132-139 */
static double* rt(orc_solver* s) { return s->prec ? s->vec[RT] : s->vec[R]; }
static double* st_(orc_solver* s) { return s->prec ? s->vec[ST] : s->vec[S]; }
static double* wt(orc_solver* s) { return s->prec ? s->vec[WT] : s->vec[W]; }
static double* ut(orc_solver* s) { return s->prec ? s->vec[UT] : s->vec[U]; }

static double* alloc_vec(orc_solver* s, int which) {
    if (!s->vec[which]) s->vec[which] = (double*)calloc((size_t)(s->n ? s->n : 1), sizeof(double));
    return s->vec[which];
}

/* the four seams of variants.cpp:107-126 */
static void apply_a(orc_solver* s, const double* in, double* out) {
    orc_spmv(s->n, s->rp, s->ci, s->va, in, out);
    s->spmv_calls++;
}
static void apply_a_block(orc_solver* s, const double* i1, const double* i2, double* o1,
                          double* o2) {
    orc_block_spmv(s->n, s->rp, s->ci, s->va, i1, i2, o1, o2);
    s->block_calls++;
}
static void apply_m(orc_solver* s, const double* in, double* out) {
    if (s->prec)
        for (int64_t i = 0; i < s->n; ++i) out[i] = s->inv_diag[i] * in[i];
    else
        memcpy(out, in, sizeof(double) * (size_t)s->n);
    s->prec_applies++;
}
static double reduce_dot(orc_solver* s, const double* x, const double* y) {
    s->reductions++;
    return orc_dot(s->n, x, y, &s->dcfg);
}

/* vector_ops.hpp:32-47 */
static void add_scaled(int64_t n, double* y, double a, const double* x) {
    for (int64_t i = 0; i < n; ++i) y[i] += a * x[i];
}
static void sub_scaled(int64_t n, double* y, double a, const double* x) {
    for (int64_t i = 0; i < n; ++i) y[i] -= a * x[i];
}
static void xpby(int64_t n, double* y, double b, const double* x) {
    for (int64_t i = 0; i < n; ++i) y[i] = x[i] + b * y[i];
}

/* variants.cpp:128-173 */
static void fail(orc_solver* s, int reason) {
    s->state = ST_BREAKDOWN;
    s->reason = reason;
}
static int settle_nonpositive(orc_solver* s, double value, int reason) {
    if (!isfinite(value)) {
        fail(s, BR_NONFINITE);
        return 1;
    }
    if (value > 0.0) return 0;
    if (value == 0.0 && orc_dot(s->n, s->vec[R], s->vec[R], &s->dcfg) == 0.0) {
        s->state = ST_CONVERGED;
        s->criterion = CB_ZERO;
    } else {
        fail(s, reason);
    }
    return 1;
}
static int settle_mu(orc_solver* s) {
    if (!isfinite(s->mu)) {
        fail(s, BR_NONFINITE);
        return 1;
    }
    if (s->mu <= 0.0) {
        fail(s, BR_MU);
        return 1;
    }
    return 0;
}
static int finalize_alpha(orc_solver* s) {
    s->alpha = s->nu / s->mu;
    if (!isfinite(s->alpha) || !isfinite(s->beta)) {
        fail(s, BR_NONFINITE);
        return 1;
    }
    return 0;
}

/* variants.cpp:175-187 */
static double predicted_nu(const orc_solver* s) {
    switch (s->nu_expr) {
        case NU_SIMPLIFIED: return s->nu - 2.0 * s->alpha * s->delta + s->alpha * s->alpha * s->gamma;
        case NU_MEURANT: return -s->nu + s->alpha * s->alpha * s->gamma;
        default:
            return s->nu - s->alpha * (s->delta + s->delta_hat) + s->alpha * s->alpha * s->gamma;
    }
}

/* variants.cpp:189-205 (paper Alg. 1) */
static void step_hs(orc_solver* s) {
    const int64_t n = s->n;
    add_scaled(n, s->vec[X], s->alpha, s->vec[P]);
    sub_scaled(n, s->vec[R], s->alpha, s->vec[S]);
    if (s->prec) apply_m(s, s->vec[R], s->vec[RT]);
    const double nu_next = reduce_dot(s, rt(s), s->vec[R]);
    if (settle_nonpositive(s, nu_next, BR_NU)) {
        s->nu = nu_next;
        return;
    }
    s->beta = nu_next / s->nu;
    s->nu = nu_next;
    xpby(n, s->vec[P], s->beta, rt(s));
    apply_a(s, s->vec[P], s->vec[S]);
    s->mu = reduce_dot(s, s->vec[P], s->vec[S]);
    if (settle_mu(s)) return;
    finalize_alpha(s);
}

/* variants.cpp:207-234 */
static void step_cg_cg(orc_solver* s) {
    const int64_t n = s->n;
    add_scaled(n, s->vec[X], s->alpha, s->vec[P]);
    sub_scaled(n, s->vec[R], s->alpha, s->vec[S]);
    if (s->prec) apply_m(s, s->vec[R], s->vec[RT]);
    apply_a(s, rt(s), s->vec[W]);
    const double nu_next = reduce_dot(s, rt(s), s->vec[R]);
    s->eta = reduce_dot(s, rt(s), s->vec[W]);
    if (settle_nonpositive(s, nu_next, BR_NU)) {
        s->nu = nu_next;
        return;
    }
    s->beta = nu_next / s->nu;
    double d_rs = 0.0, d_pw = 0.0;
    if (s->unsimplified_mu) {
        d_rs = reduce_dot(s, rt(s), s->vec[S]);
        d_pw = reduce_dot(s, s->vec[P], s->vec[W]);
    }
    const double mu_prev = s->mu;
    s->nu = nu_next;
    xpby(n, s->vec[P], s->beta, rt(s));
    xpby(n, s->vec[S], s->beta, s->vec[W]);
    s->mu = s->unsimplified_mu ? s->eta + s->beta * (d_rs + d_pw) + s->beta * s->beta * mu_prev
                               : s->eta - (s->beta / s->alpha) * s->nu;
    if (settle_mu(s)) return;
    finalize_alpha(s);
}

/* variants.cpp:237-265 (PR, paper Alg. 2; M with the Meurant expression) */
static void step_pr(orc_solver* s) {
    const int64_t n = s->n;
    add_scaled(n, s->vec[X], s->alpha, s->vec[P]);
    sub_scaled(n, s->vec[R], s->alpha, s->vec[S]);
    if (s->prec) sub_scaled(n, s->vec[RT], s->alpha, s->vec[ST]);
    s->nu_prime = predicted_nu(s);
    if (settle_nonpositive(s, s->nu_prime, BR_NUPRIME)) return;
    s->beta = s->nu_prime / s->nu;
    xpby(n, s->vec[P], s->beta, rt(s));
    apply_a(s, s->vec[P], s->vec[S]);
    if (s->prec) apply_m(s, s->vec[S], s->vec[ST]);
    s->mu = reduce_dot(s, s->vec[P], s->vec[S]);
    if (s->nu_expr != NU_MEURANT || s->track_delta) s->delta = reduce_dot(s, rt(s), s->vec[S]);
    if (s->nu_expr == NU_EXPANDED) s->delta_hat = reduce_dot(s, st_(s), s->vec[R]);
    s->gamma = reduce_dot(s, st_(s), s->vec[S]);
    if (settle_mu(s)) return;
    if (s->recompute_nu) {
        const double nu_next = reduce_dot(s, rt(s), s->vec[R]);
        if (settle_nonpositive(s, nu_next, BR_NU)) {
            s->nu = nu_next;
            return;
        }
        s->nu = nu_next;
    } else {
        s->nu = s->nu_prime;
    }
    finalize_alpha(s);
}

/* variants.cpp:267-298 */
static void step_gv(orc_solver* s) {
    const int64_t n = s->n;
    add_scaled(n, s->vec[X], s->alpha, s->vec[P]);
    sub_scaled(n, s->vec[R], s->alpha, s->vec[S]);
    if (s->prec) sub_scaled(n, s->vec[RT], s->alpha, s->vec[ST]);
    sub_scaled(n, s->vec[W], s->alpha, s->vec[U]);
    if (s->prec) apply_m(s, s->vec[W], s->vec[WT]);
    const double nu_next = reduce_dot(s, rt(s), s->vec[R]);
    s->eta = reduce_dot(s, rt(s), s->vec[W]);
    apply_a(s, wt(s), s->vec[T]);
    if (settle_nonpositive(s, nu_next, BR_NU)) {
        s->nu = nu_next;
        return;
    }
    s->beta = nu_next / s->nu;
    double d_rs = 0.0, d_pw = 0.0;
    if (s->unsimplified_mu) {
        d_rs = reduce_dot(s, rt(s), s->vec[S]);
        d_pw = reduce_dot(s, s->vec[P], s->vec[W]);
    }
    const double mu_prev = s->mu;
    s->nu = nu_next;
    xpby(n, s->vec[P], s->beta, rt(s));
    xpby(n, s->vec[S], s->beta, s->vec[W]);
    if (s->prec) xpby(n, s->vec[ST], s->beta, s->vec[WT]);
    xpby(n, s->vec[U], s->beta, s->vec[T]);
    s->mu = s->unsimplified_mu ? s->eta + s->beta * (d_rs + d_pw) + s->beta * s->beta * mu_prev
                               : s->eta - (s->beta / s->alpha) * s->nu;
    if (settle_mu(s)) return;
    finalize_alpha(s);
}

/* variants.cpp:303-350 (pipe-PR, paper Alg. 3; pipe-PR-M with Meurant) */
static void step_pipe_pr(orc_solver* s) {
    const int64_t n = s->n;
    s->nu_prime = predicted_nu(s);
    const double beta_next = s->nu_prime / s->nu;
    add_scaled(n, s->vec[X], s->alpha, s->vec[P]);
    sub_scaled(n, s->vec[R], s->alpha, s->vec[S]);
    if (s->prec) sub_scaled(n, s->vec[RT], s->alpha, s->vec[ST]);
    sub_scaled(n, s->vec[W], s->alpha, s->vec[U]);
    if (s->prec) sub_scaled(n, s->vec[WT], s->alpha, s->vec[UT]);
    if (settle_nonpositive(s, s->nu_prime, BR_NUPRIME)) return;
    s->beta = beta_next;
    xpby(n, s->vec[P], s->beta, rt(s));
    xpby(n, s->vec[S], s->beta, s->vec[W]);
    if (s->prec) xpby(n, s->vec[ST], s->beta, s->vec[WT]);
    if (s->recompute_w) {
        apply_a_block(s, st_(s), rt(s), s->vec[U], s->vec[W]);
        if (s->prec) {
            apply_m(s, s->vec[U], s->vec[UT]);
            apply_m(s, s->vec[W], s->vec[WT]);
        }
    } else {
        apply_a(s, st_(s), s->vec[U]);
        if (s->prec) apply_m(s, s->vec[U], s->vec[UT]);
    }
    s->mu = reduce_dot(s, s->vec[P], s->vec[S]);
    if (s->nu_expr != NU_MEURANT || s->track_delta) s->delta = reduce_dot(s, rt(s), s->vec[S]);
    if (s->nu_expr == NU_EXPANDED) s->delta_hat = reduce_dot(s, st_(s), s->vec[R]);
    s->gamma = reduce_dot(s, st_(s), s->vec[S]);
    if (settle_mu(s)) return;
    if (s->recompute_nu) {
        const double nu_next = reduce_dot(s, rt(s), s->vec[R]);
        if (settle_nonpositive(s, nu_next, BR_NU)) {
            s->nu = nu_next;
            return;
        }
        s->nu = nu_next;
    } else {
        s->nu = s->nu_prime;
    }
    finalize_alpha(s);
}

/* variants.cpp:354-444 (paper Appendix C "Initializations") */
static void initialize(orc_solver* s, const double* b, const double* x0) {
    const int64_t n = s->n;
    const int v = s->variant;
    const int needs_st = s->prec && v != V_HS && v != V_CG_CG;
    memcpy(alloc_vec(s, X), x0, sizeof(double) * (size_t)n);
    alloc_vec(s, R);
    apply_a(s, s->vec[X], s->vec[R]);
    for (int64_t i = 0; i < n; ++i) s->vec[R][i] = b[i] - s->vec[R][i];
    if (s->prec) apply_m(s, s->vec[R], alloc_vec(s, RT));
    s->nu = reduce_dot(s, rt(s), s->vec[R]);
    if (settle_nonpositive(s, s->nu, BR_NU)) return;
    memcpy(alloc_vec(s, P), rt(s), sizeof(double) * (size_t)n);
    alloc_vec(s, S);
    apply_a(s, s->vec[P], s->vec[S]);
    s->mu = reduce_dot(s, s->vec[P], s->vec[S]);
    if (settle_mu(s)) return;
    s->alpha = s->nu / s->mu;
    if (needs_st) apply_m(s, s->vec[S], alloc_vec(s, ST));
    switch (v) {
        case V_HS: break;
        case V_CG_CG: alloc_vec(s, W); break;
        case V_M:
        case V_PR:
            if (v == V_PR || s->nu_expr != NU_MEURANT || s->track_delta)
                s->delta = reduce_dot(s, rt(s), s->vec[S]);
            if (s->nu_expr == NU_EXPANDED) s->delta_hat = reduce_dot(s, st_(s), s->vec[R]);
            s->gamma = reduce_dot(s, st_(s), s->vec[S]);
            break;
        case V_GV:
            apply_a(s, rt(s), alloc_vec(s, W));
            apply_a(s, st_(s), alloc_vec(s, U));
            alloc_vec(s, T);
            if (s->prec) alloc_vec(s, WT);
            break;
        default: /* pipelined PR */
            apply_a(s, rt(s), alloc_vec(s, W));
            if (s->prec) apply_m(s, s->vec[W], alloc_vec(s, WT));
            apply_a(s, st_(s), alloc_vec(s, U));
            if (s->prec) apply_m(s, s->vec[U], alloc_vec(s, UT));
            if (s->nu_expr != NU_MEURANT || s->track_delta)
                s->delta = reduce_dot(s, rt(s), s->vec[S]);
            if (s->nu_expr == NU_EXPANDED) s->delta_hat = reduce_dot(s, st_(s), s->vec[R]);
            s->gamma = reduce_dot(s, st_(s), s->vec[S]);
            break;
    }
}

orc_solver* orc_solver_create(int64_t n, const int64_t* rp, const int64_t* ci,
                              const double* v, int variant, int nu_expr, int recompute_nu,
                              int recompute_w, int unsimplified_mu, int track_delta,
                              int precond, const double* b, const double* x0,
                              const orc_dotcfg* dcfg, int* err) {
    *err = 0;
    if (nu_expr < 0) nu_expr = (variant == V_M || variant == V_PIPE_PR_M) ? NU_MEURANT : NU_SIMPLIFIED;
    if (orc_config_validate(variant, nu_expr, recompute_nu, recompute_w, unsimplified_mu,
                            track_delta) != 0) {
        *err = -1;
        return NULL;
    }
    orc_solver* s = (orc_solver*)calloc(1, sizeof(orc_solver));
    s->n = n;
    s->rp = rp;
    s->ci = ci;
    s->va = v;
    s->variant = variant;
    s->nu_expr = nu_expr;
    s->recompute_nu = recompute_nu;
    s->recompute_w = recompute_w;
    s->unsimplified_mu = unsimplified_mu;
    s->track_delta = track_delta;
    s->prec = precond != 0;
    if (dcfg) s->dcfg = *dcfg;
    if (s->dcfg.mode == ORC_DOT_PART) {
        for (int p = 0; p <= s->dcfg.nparts && p < 65; ++p) s->part_copy[p] = dcfg->part_lo[p];
        s->dcfg.part_lo = s->part_copy;
    }
    if (s->prec) {
        s->inv_diag = (double*)malloc(sizeof(double) * (size_t)(n ? n : 1));
        if (orc_jacobi(n, rp, ci, v, s->inv_diag) != 0) {
            *err = -1;
            orc_solver_destroy(s);
            return NULL;
        }
    }
    initialize(s, b, x0);
    return s;
}

void orc_solver_destroy(orc_solver* s) {
    if (!s) return;
    for (int i = 0; i < 11; ++i) free(s->vec[i]);
    free(s->inv_diag);
    free(s);
}

/* variants.cpp:446-458 */
int orc_solver_step(orc_solver* s) {
    if (s->state != ST_RUNNING) return -2;
    s->k++;
    switch (s->variant) {
        case V_HS: step_hs(s); break;
        case V_CG_CG: step_cg_cg(s); break;
        case V_M:
        case V_PR: step_pr(s); break;
        case V_GV: step_gv(s); break;
        default: step_pipe_pr(s); break;
    }
    return 0;
}

void orc_solver_state(const orc_solver* s, int* k, int* status4, double* sc, uint64_t* stats4) {
    *k = s->k;
    status4[0] = s->state;
    status4[1] = s->reason;
    status4[2] = s->criterion;
    int cnt = 0;
    for (int i = 0; i < 11; ++i) cnt += s->vec[i] != NULL;
    status4[3] = cnt;
    sc[0] = s->alpha; sc[1] = s->beta; sc[2] = s->nu; sc[3] = s->nu_prime; sc[4] = s->mu;
    sc[5] = s->delta; sc[6] = s->delta_hat; sc[7] = s->gamma; sc[8] = s->eta;
    stats4[0] = s->spmv_calls;
    stats4[1] = s->block_calls;
    stats4[2] = s->prec_applies;
    stats4[3] = s->reductions;
}

int orc_solver_vector(const orc_solver* s, int which, double* out) {
    if (which < 0 || which > 10 || !s->vec[which]) return -1;
    memcpy(out, s->vec[which], sizeof(double) * (size_t)s->n);
    return 0;
}

static double true_res(orc_solver* s, const double* b, double* tmp) {
    orc_spmv(s->n, s->rp, s->ci, s->va, s->vec[X], tmp);
    for (int64_t i = 0; i < s->n; ++i) tmp[i] = b[i] - tmp[i];
    return sqrt(orc_dot(s->n, tmp, tmp, &s->dcfg));
}

/* the parity driver: same protocol as cgvref_solve in ref_shim.cpp */
int orc_solve(orc_solver* s, const double* b, int max_iter, double tol, double* upd_hist,
              double* true_hist, int true_cap) {
    double* tmp = (double*)malloc(sizeof(double) * (size_t)(s->n ? s->n : 1));
    const double bnorm = sqrt(orc_dot(s->n, b, b, &s->dcfg));
    upd_hist[0] = sqrt(orc_dot(s->n, s->vec[R], s->vec[R], &s->dcfg));
    if (true_cap > 0) true_hist[0] = true_res(s, b, tmp);
    int taken = 0;
    while (s->state == ST_RUNNING && taken < max_iter) {
        orc_solver_step(s);
        ++taken;
        const double upd = sqrt(orc_dot(s->n, s->vec[R], s->vec[R], &s->dcfg));
        upd_hist[taken] = upd;
        if (taken < true_cap) true_hist[taken] = true_res(s, b, tmp);
        if (tol > 0.0 && upd <= tol * bnorm) break;
    }
    free(tmp);
    return taken;
}

double orc_time_steps(orc_solver* s, int iters, int* taken) {
    struct timespec t0, t1;
    clock_gettime(CLOCK_MONOTONIC, &t0);
    int k = 0;
    for (; k < iters && s->state == ST_RUNNING; ++k) orc_solver_step(s);
    clock_gettime(CLOCK_MONOTONIC, &t1);
    *taken = k;
    return (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
}

/* a_norm with the clamp of src/sparse_matrix.cpp:169-178 (sequential dot, as
 * the reference's diagnostics use) */
static double a_norm_seq(const orc_solver* s, const double* e, double* tmp) {
    orc_spmv(s->n, s->rp, s->ci, s->va, e, tmp);
    double q = dot_seq(s->n, e, tmp);
    if (q < 0.0) q = 0.0;
    return sqrt(q);
}

/* The Table-3 protocol: run() with StopRule::error_reduction(threshold) and
 * per-iteration probes (src/runner.cpp:32-147, summarize in
 * src/diagnostics.cpp:111-126): the relative A-norm error after every step;
 * iters_to_1e5 = first k with ratio < 1e-5 (-1 if none); min_log10_err over
 * k >= 0. threshold <= 0: fixed budget. Returns the steps taken. */
int orc_anorm_run(orc_solver* s, const double* x_star, int max_iter, double threshold,
                  int* iters_to_1e5, double* min_log10_err, int* final_state) {
    const int64_t n = s->n;
    double* e = (double*)malloc(sizeof(double) * (size_t)(n ? n : 1));
    double* tmp = (double*)malloc(sizeof(double) * (size_t)(n ? n : 1));
    for (int64_t i = 0; i < n; ++i) e[i] = x_star[i] - s->vec[X][i];
    const double e0 = a_norm_seq(s, e, tmp);
    double min_ratio = 1.0; /* k = 0 record: ratio 1 */
    *iters_to_1e5 = -1;
    int taken = 0, stopped = 0;
    while (s->state == ST_RUNNING && taken < max_iter) {
        orc_solver_step(s);
        ++taken;
        for (int64_t i = 0; i < n; ++i) e[i] = x_star[i] - s->vec[X][i];
        const double ratio = a_norm_seq(s, e, tmp) / e0;
        if (ratio < min_ratio) min_ratio = ratio;
        if (*iters_to_1e5 < 0 && ratio < 1e-5) *iters_to_1e5 = s->k;
        if (threshold > 0.0 && ratio < threshold && s->state == ST_RUNNING) {
            stopped = 1;
            break;
        }
    }
    *min_log10_err = log10(min_ratio);
    *final_state = stopped ? ST_CONVERGED : (s->state == ST_RUNNING ? ST_MAXITER : s->state);
    free(e);
    free(tmp);
    return taken;
}
