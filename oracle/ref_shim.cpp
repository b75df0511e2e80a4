// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the UNCHANGED reference sources
// (/root/reference/proj/src/{variants,sparse_matrix,preconditioner,runner,
//  diagnostics,matrix_market}.cpp), compiled with -Dcgv=cgv_ref
// -ffp-contract=off by oracle/Makefile into oracle/_ref/libcgvref.so.
//
// It exists so that Python tests, the golden-vector script and bench.py's
// reference arm can drive the reference's own solver:
//   initialize / step      proj/include/cgvariants/variants.hpp:149-153
//   run                    proj/include/cgvariants/runner.hpp:47-49
//   spmv / block_spmv      proj/include/cgvariants/sparse_matrix.hpp:41-47
//   Preconditioner         proj/include/cgvariants/preconditioner.hpp:13-28
//   parse Matrix Market    proj/include/cgvariants/matrix_market.hpp:32-38
// Only reference headers are included; no reference code is copied here.
#include "cgvariants/diagnostics.hpp"
#include "cgvariants/matrix_market.hpp"
#include "cgvariants/preconditioner.hpp"
#include "cgvariants/runner.hpp"
#include "cgvariants/sparse_matrix.hpp"
#include "cgvariants/variants.hpp"
#include "cgvariants/vector_ops.hpp"

#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>

using namespace cgv;  // renamed to cgv_ref by -Dcgv=cgv_ref

namespace {

thread_local std::string g_err;

int fail_with(const std::exception& e, int code) {
    g_err = e.what();
    return code;
}

// error codes mirror include/cgvk.h: -1 invalid_argument, -2 logic_error, -9 other
int classify(const std::exception_ptr& p) {
    try {
        std::rethrow_exception(p);
    } catch (const std::invalid_argument& e) {
        return fail_with(e, -1);
    } catch (const std::logic_error& e) {
        return fail_with(e, -2);
    } catch (const std::exception& e) {
        return fail_with(e, -9);
    }
    return -9;
}

struct RefSolver {
    SparseMatrix* a;  // borrowed
    Preconditioner m;
    SolverState st;
};

VariantConfig make_config(int variant, int nu_expr, int recompute_nu, int recompute_w,
                          int unsimplified_mu, int track_delta) {
    VariantConfig c = VariantConfig::make(static_cast<Variant>(variant));
    if (nu_expr >= 0) c.nu_expression = static_cast<NuExpression>(nu_expr);
    c.recompute_nu = recompute_nu != 0;
    c.recompute_w = recompute_w != 0;
    c.unsimplified_mu = unsimplified_mu != 0;
    c.track_delta = track_delta != 0;
    return c;
}

DenseVector* vec_of(SolverState& st, int which) {
    switch (which) {
        case 0: return &st.x;
        case 1: return &st.r;
        case 2: return &st.p;
        case 3: return &st.s;
        case 4: return &st.w;
        case 5: return &st.u;
        case 6: return &st.t;
        case 7: return &st.r_tilde;
        case 8: return &st.s_tilde;
        case 9: return &st.w_tilde;
        case 10: return &st.u_tilde;
    }
    return nullptr;
}

}  // namespace

extern "C" {

const char* cgvref_last_error(void) { return g_err.c_str(); }

void* cgvref_matrix_create(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                           const double* values) {
    auto* a = new SparseMatrix;
    a->n = n;
    a->row_ptr.assign(row_ptr, row_ptr + n + 1);
    const int64_t nnz = row_ptr[n];
    a->col_idx.assign(col_idx, col_idx + nnz);
    a->values.assign(values, values + nnz);
    return a;
}

void cgvref_matrix_destroy(void* a) { delete static_cast<SparseMatrix*>(a); }

int64_t cgvref_matrix_nnz(void* a) { return static_cast<SparseMatrix*>(a)->nnz(); }

void cgvref_matrix_arrays(void* a, int64_t* row_ptr, int64_t* col_idx, double* values) {
    auto* m = static_cast<SparseMatrix*>(a);
    std::memcpy(row_ptr, m->row_ptr.data(), sizeof(int64_t) * m->row_ptr.size());
    std::memcpy(col_idx, m->col_idx.data(), sizeof(int64_t) * m->col_idx.size());
    std::memcpy(values, m->values.data(), sizeof(double) * m->values.size());
}

int64_t cgvref_matrix_n(void* a) { return static_cast<SparseMatrix*>(a)->n; }

// Matrix Market parse (the reference parser, src/matrix_market.cpp:124-202)
void* cgvref_read_mtx(const char* path) {
    try {
        return new SparseMatrix(read_matrix_market_file(path));
    } catch (...) {
        classify(std::current_exception());
        return nullptr;
    }
}

int cgvref_validate_csr(void* a) {
    try {
        validate_csr(*static_cast<SparseMatrix*>(a));
        return 0;
    } catch (...) {
        return classify(std::current_exception());
    }
}

int cgvref_is_symmetric(void* a) { return is_symmetric(*static_cast<SparseMatrix*>(a)) ? 1 : 0; }

int cgvref_spmv(void* a, const double* x, double* y) {
    auto* m = static_cast<SparseMatrix*>(a);
    try {
        spmv(*m, std::span<const double>(x, m->n), std::span<double>(y, m->n));
        return 0;
    } catch (...) {
        return classify(std::current_exception());
    }
}

int cgvref_block_spmv(void* a, const double* x1, const double* x2, double* y1, double* y2) {
    auto* m = static_cast<SparseMatrix*>(a);
    const auto n = static_cast<std::size_t>(m->n);
    try {
        block_spmv(*m, {x1, n}, {x2, n}, {y1, n}, {y2, n});
        return 0;
    } catch (...) {
        return classify(std::current_exception());
    }
}

int cgvref_jacobi(void* a, double* inv_diag) {
    try {
        Preconditioner p = Preconditioner::jacobi(*static_cast<SparseMatrix*>(a));
        std::memcpy(inv_diag, p.inv_diag.data(), sizeof(double) * p.inv_diag.size());
        return 0;
    } catch (...) {
        return classify(std::current_exception());
    }
}

double cgvref_dot(int64_t n, const double* x, const double* y) {
    return dot(std::span<const double>(x, n), std::span<const double>(y, n));
}

int cgvref_config_validate(int variant, int nu_expr, int recompute_nu, int recompute_w,
                           int unsimplified_mu, int track_delta) {
    try {
        make_config(variant, nu_expr, recompute_nu, recompute_w, unsimplified_mu, track_delta)
            .validate();
        return 0;
    } catch (...) {
        return classify(std::current_exception());
    }
}

// initialize(); returns nullptr (and sets the error) when the reference throws.
void* cgvref_solver_create(void* a, int variant, int nu_expr, int recompute_nu,
                           int recompute_w, int unsimplified_mu, int track_delta, int precond,
                           const double* b, const double* x0, int* err_code) {
    auto* m = static_cast<SparseMatrix*>(a);
    auto* s = new RefSolver;
    s->a = m;
    *err_code = 0;
    try {
        s->m = precond ? Preconditioner::jacobi(*m) : Preconditioner::identity();
        const auto n = static_cast<std::size_t>(m->n);
        DenseVector bv(b, b + n), xv(x0, x0 + n);
        s->st = initialize(make_config(variant, nu_expr, recompute_nu, recompute_w,
                                       unsimplified_mu, track_delta),
                           *m, s->m, bv, xv);
    } catch (...) {
        *err_code = classify(std::current_exception());
        delete s;
        return nullptr;
    }
    return s;
}

void cgvref_solver_destroy(void* s) { delete static_cast<RefSolver*>(s); }

int cgvref_solver_step(void* sp) {
    auto* s = static_cast<RefSolver*>(sp);
    try {
        step(s->st);
        return 0;
    } catch (...) {
        return classify(std::current_exception());
    }
}

// scalars: alpha beta nu nu_prime mu delta delta_hat gamma eta
void cgvref_solver_state(void* sp, int* k, int* status4, double* scalars9, uint64_t* stats4) {
    auto& st = static_cast<RefSolver*>(sp)->st;
    *k = st.k;
    status4[0] = static_cast<int>(st.status.state);
    status4[1] = static_cast<int>(st.status.breakdown);
    status4[2] = static_cast<int>(st.status.criterion);
    status4[3] = st.allocated_vectors();
    const double sc[9] = {st.alpha, st.beta,      st.nu,    st.nu_prime, st.mu,
                          st.delta, st.delta_hat, st.gamma, st.eta};
    std::memcpy(scalars9, sc, sizeof sc);
    stats4[0] = st.stats.spmv_calls;
    stats4[1] = st.stats.block_spmv_calls;
    stats4[2] = st.stats.precond_applies;
    stats4[3] = st.stats.reductions;
}

// Copies a working vector; returns -1 when the variant does not allocate it.
int cgvref_solver_vector(void* sp, int which, double* out) {
    auto& st = static_cast<RefSolver*>(sp)->st;
    DenseVector* v = vec_of(st, which);
    if (!v || v->empty()) return -1;
    std::memcpy(out, v->data(), sizeof(double) * v->size());
    return 0;
}

// Parity driver: steps until ||r_k|| <= tol*||b|| (tol <= 0: never)
// or max_iter, recording ||r_k|| (sequential norm2) and, for k < true_cap, the
// true residual ||b - A x_k|| from a fresh reference spmv. Returns steps taken.
int cgvref_solve(void* sp, const double* b, int max_iter, double tol, double* upd_hist,
                 double* true_hist, int true_cap) {
    auto* s = static_cast<RefSolver*>(sp);
    auto& st = s->st;
    const auto n = static_cast<std::size_t>(st.n);
    const double bnorm = norm2(std::span<const double>(b, n));
    DenseVector ax(n), res(n);
    auto true_res = [&]() {
        spmv(*s->a, st.x, ax);
        for (std::size_t i = 0; i < n; ++i) res[i] = b[i] - ax[i];
        return norm2(res);
    };
    upd_hist[0] = norm2(st.r);
    if (true_cap > 0) true_hist[0] = true_res();
    int taken = 0;
    while (st.status.running() && taken < max_iter) {
        step(st);
        ++taken;
        const double upd = norm2(st.r);
        upd_hist[taken] = upd;
        if (taken < true_cap) true_hist[taken] = true_res();
        if (tol > 0.0 && upd <= tol * bnorm) break;
    }
    return taken;
}

double cgvref_true_residual(void* sp, const double* b) {
    auto* s = static_cast<RefSolver*>(sp);
    auto& st = s->st;
    const auto n = static_cast<std::size_t>(st.n);
    DenseVector ax(n), res(n);
    spmv(*s->a, st.x, ax);
    for (std::size_t i = 0; i < n; ++i) res[i] = b[i] - ax[i];
    return norm2(res);
}

// CPU baseline timing: only the step() loop, steady_clock.
double cgvref_time_steps(void* sp, int iters, int* taken) {
    auto& st = static_cast<RefSolver*>(sp)->st;
    const auto t0 = std::chrono::steady_clock::now();
    int k = 0;
    for (; k < iters && st.status.running(); ++k) step(st);
    const auto t1 = std::chrono::steady_clock::now();
    *taken = k;
    return std::chrono::duration<double>(t1 - t0).count();
}

// run() with the A-norm error stop rule and probes: the Table-3 protocol
// (tests/test_matrices.cpp:39-46). stop_kind: 0 fixed, 1 error-reduction,
// 2 stagnation. Outputs the summary (iters_to_1e5 or -1, min log10 error),
// final status, and the probed (k, rel_err, true_res, upd_res) per record.
int cgvref_run(void* a, int variant, int precond, const double* b, const double* x0,
               const double* x_star, int max_iter, int stop_kind, double threshold,
               int cadence, int* iters_to_1e5, double* min_log10_err, int* final_state,
               int* n_records, int rec_cap, int* rec_k, double* rec_err, double* rec_true,
               double* rec_upd) {
    auto* m = static_cast<SparseMatrix*>(a);
    try {
        const auto n = static_cast<std::size_t>(m->n);
        Preconditioner pm = precond ? Preconditioner::jacobi(*m) : Preconditioner::identity();
        DenseVector bv(b, b + n), xv(x0, x0 + n), xs(x_star, x_star + n);
        StopRule rule = stop_kind == 0   ? StopRule::fixed(max_iter)
                        : stop_kind == 1 ? StopRule::error_reduction(threshold)
                                         : StopRule::stagnation();
        ProbeOptions probe;
        probe.x_star = &xs;
        probe.cadence = cadence;
        ConvergenceHistory h = run(VariantConfig::make(static_cast<Variant>(variant)), *m, pm,
                                   bv, xv, max_iter, rule, probe);
        *final_state = static_cast<int>(h.final_status.state);
        *iters_to_1e5 = -1;
        *min_log10_err = 0.0;
        if (h.summary) {
            if (h.summary->iters_to_1e5) *iters_to_1e5 = *h.summary->iters_to_1e5;
            *min_log10_err = h.summary->min_log10_err;
        }
        int cnt = 0;
        for (const auto& rec : h.records) {
            if (cnt >= rec_cap) break;
            rec_k[cnt] = rec.k;
            rec_err[cnt] = rec.rel_err_a_norm.value_or(NAN);
            rec_true[cnt] = rec.true_res_norm.value_or(NAN);
            rec_upd[cnt] = rec.upd_res_norm.value_or(NAN);
            ++cnt;
        }
        *n_records = static_cast<int>(h.records.size());
        return 0;
    } catch (...) {
        return classify(std::current_exception());
    }
}

// run() with every IterationRecord field (proj/include/cgvariants/diagnostics.hpp:16-29)
// and the full StopRule / ProbeOptions (runner.hpp:9-45): golden fixtures for
// the device run(). Per record: k, presence mask (bit f = field f present) and
// 13 values in field order rel_err_a_norm, true_res_norm, upd_res_norm,
// residual_gap_norm, nu_gap, w_gap_norm, s_gap_norm, lanczos_res_norm,
// succ_orth, alpha, beta, nu, nu_prime.
int cgvref_run_records(void* a, int variant, int nu_expr, int recompute_nu, int recompute_w,
                       int unsimplified_mu, int track_delta, int precond, const double* b,
                       const double* x0, const double* x_star, int max_iter, int stop_kind,
                       int fixed_count, double threshold, int stag_window, double stag_improvement,
                       int probes, int cadence, int* final_status /* state, breakdown, criterion */,
                       int* has_summary, int* iters_to_1e5, double* min_log10_err, int* n_records,
                       int rec_cap, int* rec_k, unsigned* rec_mask, double* rec_vals) {
    auto* m = static_cast<SparseMatrix*>(a);
    try {
        const auto n = static_cast<std::size_t>(m->n);
        Preconditioner pm = precond ? Preconditioner::jacobi(*m) : Preconditioner::identity();
        DenseVector bv(b, b + n), xv(x0, x0 + n), xs;
        if (x_star) xs.assign(x_star, x_star + n);
        StopRule rule;
        if (stop_kind == 0) {
            rule = StopRule::fixed(fixed_count);
        } else if (stop_kind == 1) {
            rule = StopRule::error_reduction(threshold);
        } else {
            rule = StopRule::stagnation(stag_window, stag_improvement);
        }
        ProbeOptions probe;
        probe.enabled = probes != 0;
        probe.cadence = cadence;
        probe.x_star = x_star ? &xs : nullptr;
        ConvergenceHistory h = run(make_config(variant, nu_expr, recompute_nu, recompute_w,
                                               unsimplified_mu, track_delta),
                                   *m, pm, bv, xv, max_iter, rule, probe);
        final_status[0] = static_cast<int>(h.final_status.state);
        final_status[1] = static_cast<int>(h.final_status.breakdown);
        final_status[2] = static_cast<int>(h.final_status.criterion);
        *has_summary = h.summary.has_value();
        *iters_to_1e5 = -1;
        *min_log10_err = 0.0;
        if (h.summary) {
            if (h.summary->iters_to_1e5) *iters_to_1e5 = *h.summary->iters_to_1e5;
            *min_log10_err = h.summary->min_log10_err;
        }
        int cnt = 0;
        for (const auto& rec : h.records) {
            if (cnt >= rec_cap) break;
            const std::optional<double>* f[13] = {
                &rec.rel_err_a_norm, &rec.true_res_norm, &rec.upd_res_norm, &rec.residual_gap_norm,
                &rec.nu_gap, &rec.w_gap_norm, &rec.s_gap_norm, &rec.lanczos_res_norm, &rec.succ_orth,
                &rec.alpha, &rec.beta, &rec.nu, &rec.nu_prime};
            rec_k[cnt] = rec.k;
            unsigned mask = 0;
            for (int q = 0; q < 13; ++q) {
                rec_vals[cnt * 13 + q] = f[q]->value_or(0.0);
                if (f[q]->has_value()) mask |= 1u << q;
            }
            rec_mask[cnt] = mask;
            ++cnt;
        }
        *n_records = static_cast<int>(h.records.size());
        return 0;
    } catch (...) {
        return classify(std::current_exception());
    }
}

// std::mt19937_64 stream, used to pin the generators' RNG.
void cgvref_mt19937_64(uint64_t seed, int64_t count, uint64_t* out) {
    std::mt19937_64 e(seed);
    for (int64_t i = 0; i < count; ++i) out[i] = e();
}

}  // extern "C"
