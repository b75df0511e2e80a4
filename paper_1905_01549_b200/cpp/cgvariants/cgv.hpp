// cgv:: — the reference's solver API (proj/include/cgvariants/*.hpp) re-declared
// over the cgvk C ABI (include/cgvk.h), so reference callers recompile against
// the B200 path unchanged. Same names, argument meaning and error behaviour:
// CGVK_EINVAL -> std::invalid_argument, CGVK_ESTATE -> std::logic_error, other
// failures -> std::runtime_error. Header-only; link with libcgvk.so.
//
// Source-compatible additions (the reference's fields are all kept):
//   * SparseMatrix::device — the matrix resident on the GPU, uploaded on first
//     use (A is immutable after that, as the reference's sharing contract,
//     inc/variants.hpp:95-97, already requires);
//   * SolverState::device / sync_host — the device solver; with sync_host
//     (default) every step() refreshes the host vectors (parity mode); with it
//     off, run()/step_n() keep everything on the device.
#pragma once

#include "cgvk.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <cstdint>
#include <memory>
#include <mutex>
#include <numeric>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <tuple>
#include <vector>

namespace cgv {

using Index = std::int64_t;             // inc/types.hpp:8
using DenseVector = std::vector<double>;  // inc/types.hpp:9

namespace detail {
inline void check(int rc) {
    if (rc == CGVK_OK) return;
    const std::string msg = cgvk_last_error();
    if (rc == CGVK_EINVAL) throw std::invalid_argument(msg);
    if (rc == CGVK_ESTATE) throw std::logic_error(msg);
    throw std::runtime_error(msg);
}
struct MatrixHandle {
    cgvk_matrix h = nullptr;
    ~MatrixHandle() { cgvk_matrix_destroy(h); }
};
struct SolverHandle {
    cgvk_solver h = nullptr;
    ~SolverHandle() { cgvk_solver_destroy(h); }
};
}  // namespace detail

// ------------------------------------------------------------ vector ops
// inc/vector_ops.hpp:15-54 (host helpers; the solver's own dots run on the
// device in its canonical reduction order). inner_product accumulates left to
// right, init + x0*y0 + x1*y1 + ..., each product rounded (built with
// -ffp-contract=off like the reference).

inline double dot(std::span<const double> x, std::span<const double> y) {
    if (x.size() != y.size()) throw std::invalid_argument("dot: operands differ in length");
    return std::inner_product(x.begin(), x.end(), y.begin(), 0.0);
}
inline double norm2(std::span<const double> x) { return std::sqrt(dot(x, x)); }

// --------------------------------------------------------- sparse matrix
// inc/sparse_matrix.hpp:16-57

namespace detail {
// The device copy of a SparseMatrix, uploaded once under a lock (solvers on
// several threads may share one A, src/experiment.cpp:317-322). A copied
// matrix starts without one: its arrays may be edited before its first use.
struct DeviceSlot {
    std::shared_ptr<MatrixHandle> handle;
    std::unique_ptr<std::mutex> lock = std::make_unique<std::mutex>();
    DeviceSlot() = default;
    DeviceSlot(const DeviceSlot&) : lock(std::make_unique<std::mutex>()) {}
    DeviceSlot& operator=(const DeviceSlot&) {
        const std::lock_guard<std::mutex> g(*lock);
        handle.reset();
        return *this;
    }
    DeviceSlot(DeviceSlot&&) noexcept = default;
    DeviceSlot& operator=(DeviceSlot&&) noexcept = default;
};
}  // namespace detail

struct SparseMatrix {
    Index n = 0;
    std::vector<Index> row_ptr;
    std::vector<Index> col_idx;
    std::vector<double> values;
    mutable detail::DeviceSlot device;  // addition

    Index nnz() const { return static_cast<Index>(values.size()); }

    cgvk_matrix on_device(int gpu = 0) const {
        const std::lock_guard<std::mutex> g(*device.lock);
        if (!device.handle) {
            if (row_ptr.size() != static_cast<std::size_t>(n) + 1)
                throw std::invalid_argument("row_ptr length must be n+1");
            auto h = std::make_shared<detail::MatrixHandle>();
            detail::check(cgvk_matrix_create_csr(n, row_ptr.data(), col_idx.data(), values.data(),
                                                 gpu, 0, &h->h));
            device.handle = std::move(h);
        }
        return device.handle->h;
    }
};

using Triplet = std::tuple<Index, Index, double>;

// sparse_matrix.hpp:25-27: entries ordered by (row, column); repeated
// positions summed in the order they were given; sums that are exactly zero
// are not stored. Rows are bucketed with a counting pass (which keeps the
// input order inside each row), then each row's entries are ordered by
// column with a stable sort and folded.
inline SparseMatrix csr_from_triplets(Index n, std::vector<Triplet> t) {
    if (n < 0) throw std::invalid_argument("csr_from_triplets: negative dimension");
    for (const Triplet& e : t)
        if (std::get<0>(e) < 0 || std::get<0>(e) >= n || std::get<1>(e) < 0 || std::get<1>(e) >= n)
            throw std::invalid_argument("csr_from_triplets: entry outside the n x n matrix");
    const auto rows = static_cast<std::size_t>(n);
    std::vector<std::size_t> start(rows + 1, 0), order(t.size());
    for (const Triplet& e : t) ++start[static_cast<std::size_t>(std::get<0>(e)) + 1];
    std::partial_sum(start.begin(), start.end(), start.begin());
    {
        std::vector<std::size_t> fill(start.begin(), start.end() - 1);
        for (std::size_t q = 0; q < t.size(); ++q) order[fill[static_cast<std::size_t>(std::get<0>(t[q]))]++] = q;
    }
    SparseMatrix a;
    a.n = n;
    a.row_ptr.reserve(rows + 1);
    a.row_ptr.push_back(0);
    for (std::size_t r = 0; r < rows; ++r) {
        const auto first = order.begin() + static_cast<std::ptrdiff_t>(start[r]);
        const auto last = order.begin() + static_cast<std::ptrdiff_t>(start[r + 1]);
        std::stable_sort(first, last, [&t](std::size_t p, std::size_t q) { return std::get<1>(t[p]) < std::get<1>(t[q]); });
        for (auto it = first; it != last;) {
            const Index col = std::get<1>(t[*it]);
            double acc = std::get<2>(t[*it]);
            for (++it; it != last && std::get<1>(t[*it]) == col; ++it) acc += std::get<2>(t[*it]);
            if (acc == 0.0) continue;
            a.col_idx.push_back(col);
            a.values.push_back(acc);
        }
        a.row_ptr.push_back(static_cast<Index>(a.values.size()));
    }
    return a;
}

// validated on the device (cgvk_matrix_create_csr runs validate_csr there)
inline void validate_csr(const SparseMatrix& a) {
    const SparseMatrix copy{a.n, a.row_ptr, a.col_idx, a.values, {}};
    copy.on_device();
}

inline bool is_symmetric(const SparseMatrix& a) {
    cgvk_matrix h = nullptr;
    const int rc = cgvk_matrix_create_csr(a.n, a.row_ptr.data(), a.col_idx.data(), a.values.data(), 0,
                                          CGVK_MATRIX_CHECK_SYMMETRIC, &h);
    cgvk_matrix_destroy(h);
    if (rc == CGVK_EINVAL) return false;
    detail::check(rc);
    return true;
}

// y = A x, per-row left-to-right (sparse_matrix.hpp:41-42) — on the GPU
inline void spmv(const SparseMatrix& a, std::span<const double> x, std::span<double> y) {
    if (x.size() != static_cast<std::size_t>(a.n) || y.size() != static_cast<std::size_t>(a.n))
        throw std::invalid_argument("spmv dimension mismatch");
    detail::check(cgvk_spmv(a.on_device(), x.data(), y.data()));
}
inline DenseVector spmv(const SparseMatrix& a, const DenseVector& x) {
    DenseVector y(static_cast<std::size_t>(a.n));
    spmv(a, x, y);
    return y;
}
inline void block_spmv(const SparseMatrix& a, std::span<const double> x1, std::span<const double> x2,
                       std::span<double> y1, std::span<double> y2) {
    const auto n = static_cast<std::size_t>(a.n);
    if (x1.size() != n || x2.size() != n || y1.size() != n || y2.size() != n)
        throw std::invalid_argument("block_spmv dimension mismatch");
    detail::check(cgvk_block_spmv(a.on_device(), x1.data(), x2.data(), y1.data(), y2.data()));
}

// ---------------------------------------------------------- preconditioner
// inc/preconditioner.hpp:13-28

namespace detail {
inline std::uint64_t digest(const std::vector<double>& v) {
    std::uint64_t h = 0x9e3779b97f4a7c15ull;
    for (const double d : v) {
        std::uint64_t bits;
        std::memcpy(&bits, &d, sizeof bits);
        h = (h ^ bits) * 0x100000001b3ull;
    }
    return h;
}
}  // namespace detail

// The device solver applies Jacobi as 1/diag(A) of the solver's own matrix
// (recomputed there bit-identically to Preconditioner::jacobi). A Jacobi
// preconditioner is therefore accepted only for the matrix it was built from
// and with inv_diag as built; anything else is rejected with
// std::invalid_argument rather than silently solving a different system
// (INTEGRATION.md §3).
struct Preconditioner {
    enum class Kind { Identity, Jacobi };
    Kind kind = Kind::Identity;
    std::vector<double> inv_diag;
    const SparseMatrix* source = nullptr;  // addition: the matrix it was built from
    std::uint64_t built_digest = 0;        // addition: digest(inv_diag) at construction

    static Preconditioner identity() { return Preconditioner{}; }
    static Preconditioner jacobi(const SparseMatrix& a) {
        Preconditioner m;
        m.kind = Kind::Jacobi;
        m.source = &a;
        m.inv_diag.resize(static_cast<std::size_t>(a.n));
        detail::check(cgvk_jacobi(a.on_device(), m.inv_diag.data()));
        m.built_digest = detail::digest(m.inv_diag);
        return m;
    }
    // CGVK_PRECOND_* for a solve with `a`; throws when the device would not
    // apply exactly this preconditioner.
    int device_kind_for(const SparseMatrix& a) const {
        if (kind == Kind::Identity) return CGVK_PRECOND_IDENTITY;
        if (inv_diag.size() != static_cast<std::size_t>(a.n))
            throw std::invalid_argument("preconditioner dimension mismatch");
        if (source != &a)
            throw std::invalid_argument("Jacobi preconditioner was built from a different matrix");
        if (detail::digest(inv_diag) != built_digest)
            throw std::invalid_argument("Jacobi inv_diag was modified after construction");
        return CGVK_PRECOND_JACOBI;
    }
    void apply(std::span<const double> in, std::span<double> out) const {
        if (in.size() != out.size()) throw std::invalid_argument("preconditioner dimension mismatch");
        if (kind == Kind::Identity) {
            std::copy(in.begin(), in.end(), out.begin());
            return;
        }
        if (in.size() != inv_diag.size()) throw std::invalid_argument("preconditioner dimension mismatch");
        for (std::size_t i = 0; i < in.size(); ++i) out[i] = inv_diag[i] * in[i];
    }
    DenseVector apply(const DenseVector& in) const {
        DenseVector out(in.size());
        apply(in, out);
        return out;
    }
    bool is_identity() const { return kind == Kind::Identity; }
};

inline std::string_view preconditioner_name(Preconditioner::Kind k) {
    return k == Preconditioner::Kind::Identity ? "none" : "jacobi";
}

// ---------------------------------------------------------------- variants
// inc/variants.hpp:17-153

enum class Variant { HS, CG_CG, M, PR, GV, PIPE_PR_M, PIPE_PR };
enum class NuExpression { Expanded, Simplified, Meurant };

struct VariantConfig {
    Variant variant = Variant::HS;
    bool recompute_nu = true;
    bool recompute_w = true;
    NuExpression nu_expression = NuExpression::Simplified;
    bool unsimplified_mu = false;
    bool track_delta = false;

    static VariantConfig make(Variant v) {
        const cgvk_variant_config c = cgvk_variant_config_make(static_cast<int>(v));
        VariantConfig out;
        out.variant = v;
        out.nu_expression = static_cast<NuExpression>(c.nu_expression);
        return out;
    }
    cgvk_variant_config to_c() const {
        return {static_cast<int>(variant), static_cast<int>(nu_expression), recompute_nu, recompute_w,
                unsimplified_mu, track_delta};
    }
    void validate() const {
        const cgvk_variant_config c = to_c();
        detail::check(cgvk_variant_config_validate(&c));
    }
    bool is_predictor() const {
        return variant == Variant::M || variant == Variant::PR || variant == Variant::PIPE_PR_M ||
               variant == Variant::PIPE_PR;
    }
    bool is_pipelined() const {
        return variant == Variant::GV || variant == Variant::PIPE_PR_M || variant == Variant::PIPE_PR;
    }
};

inline std::string_view variant_name(Variant v) {
    constexpr std::string_view names[] = {"hs", "cg", "m", "pr", "gv", "pipe-pr-m", "pipe-pr"};
    return names[static_cast<int>(v)];
}

enum class BreakdownReason { None, NuPrimeNonPositive, NuNonPositive, MuNonPositive, NonFinite };
enum class ConvergedBy { ZeroResidual, ErrorThreshold, Stagnation, Tolerance };

struct SolveStatus {
    enum class State { Running, Breakdown, MaxIterations, Converged };
    State state = State::Running;
    BreakdownReason breakdown = BreakdownReason::None;
    ConvergedBy criterion = ConvergedBy::ZeroResidual;
    bool running() const { return state == State::Running; }
};

struct SolverStats {
    std::uint64_t spmv_calls = 0, block_spmv_calls = 0, precond_applies = 0, reductions = 0;
};

struct SolverState {
    VariantConfig config;
    const SparseMatrix* a = nullptr;
    const Preconditioner* m = nullptr;
    bool preconditioned = false;
    Index n = 0;
    int k = 0;
    SolveStatus status;
    SolverStats stats;
    DenseVector x, r, p, s, w, u, t, r_tilde, s_tilde, w_tilde, u_tilde;
    double alpha = 0.0, beta = 0.0, nu = 0.0, nu_prime = 0.0, mu = 0.0, delta = 0.0,
           delta_hat = 0.0, gamma = 0.0, eta = 0.0;
    // additions
    std::shared_ptr<detail::SolverHandle> device;
    bool sync_host = true;

    DenseVector& rt() { return preconditioned ? r_tilde : r; }
    DenseVector& st() { return preconditioned ? s_tilde : s; }
    DenseVector& wt() { return preconditioned ? w_tilde : w; }
    DenseVector& ut() { return preconditioned ? u_tilde : u; }
    int allocated_vectors() const {
        int c = 0;
        for (const DenseVector* v : {&x, &r, &p, &s, &w, &u, &t, &r_tilde, &s_tilde, &w_tilde, &u_tilde})
            c += !v->empty();
        return c;
    }

    // Pull status, scalars, counters (and the vectors when sync_host) from the device.
    void refresh() {
        cgvk_solve_status st{};
        cgvk_scalars sc{};
        cgvk_stats ss{};
        detail::check(cgvk_solver_status(device->h, &st, &sc, &ss));
        k = st.k;
        status.state = static_cast<SolveStatus::State>(st.state);
        status.breakdown = static_cast<BreakdownReason>(st.breakdown);
        status.criterion = static_cast<ConvergedBy>(st.criterion);
        alpha = sc.alpha;
        beta = sc.beta;
        nu = sc.nu;
        nu_prime = sc.nu_prime;
        mu = sc.mu;
        delta = sc.delta;
        delta_hat = sc.delta_hat;
        gamma = sc.gamma;
        eta = sc.eta;
        stats = {ss.spmv_calls, ss.block_spmv_calls, ss.precond_applies, ss.reductions};
        if (!sync_host) return;
        DenseVector* vecs[] = {&x, &r, &p, &s, &w, &u, &t, &r_tilde, &s_tilde, &w_tilde, &u_tilde};
        for (int which = 0; which < 11; ++which) {
            DenseVector& v = *vecs[which];
            v.resize(static_cast<std::size_t>(n));
            if (n == 0 || cgvk_solver_get_vector(device->h, which, v.data()) != CGVK_OK) v.clear();
        }
    }
};

// initialize() (inc/variants.hpp:149-150)
inline SolverState initialize(const VariantConfig& config, const SparseMatrix& a,
                              const Preconditioner& m, const DenseVector& b, const DenseVector& x0) {
    config.validate();
    if (b.size() != static_cast<std::size_t>(a.n) || x0.size() != static_cast<std::size_t>(a.n))
        throw std::invalid_argument("right-hand side or initial guess dimension mismatch");
    const int precond = m.device_kind_for(a);
    SolverState st;
    st.config = config;
    st.a = &a;
    st.m = &m;
    st.preconditioned = !m.is_identity();
    st.n = a.n;
    st.device = std::make_shared<detail::SolverHandle>();
    const cgvk_variant_config c = config.to_c();
    detail::check(cgvk_solver_create(a.on_device(), &c, precond, b.data(), x0.data(), &st.device->h));
    st.refresh();
    return st;
}

// step() (inc/variants.hpp:153): exactly one iteration
inline void step(SolverState& st) {
    if (!st.status.running()) throw std::logic_error("step() on a terminated solver");
    detail::check(cgvk_solver_step(st.device->h, 1));
    detail::check(cgvk_solver_sync(st.device->h));
    st.refresh();
}

// Performance entry: n iterations as graph replays, one sync at the end.
inline void step_n(SolverState& st, int n_iters, double rel_tol = 0.0) {
    if (!st.status.running()) throw std::logic_error("step() on a terminated solver");
    if (rel_tol > 0.0) detail::check(cgvk_solver_set_tolerance(st.device->h, rel_tol));
    detail::check(cgvk_solver_step(st.device->h, n_iters));
    detail::check(cgvk_solver_sync(st.device->h));
    st.refresh();
}

// ------------------------------------------------------------------ runner
// inc/runner.hpp + inc/diagnostics.hpp: StopRule, ProbeOptions,
// IterationRecord, Summary, ConvergenceHistory, run() — the whole driver runs
// on the device (cgvk_run): every probe quantity from fresh device products.

struct StopRule {
    enum class Kind { FixedIterations, ErrorReduction, ResidualStagnation };
    Kind kind = Kind::ResidualStagnation;
    int fixed_count = 0;
    double error_threshold = 1e-5;
    int stagnation_window = 50;
    double stagnation_improvement = 0.01;
    static StopRule fixed(int count) {
        StopRule r;
        r.kind = Kind::FixedIterations;
        r.fixed_count = count;
        return r;
    }
    static StopRule error_reduction(double threshold) {
        StopRule r;
        r.kind = Kind::ErrorReduction;
        r.error_threshold = threshold;
        return r;
    }
    static StopRule stagnation(int window = 50, double improvement = 0.01) {
        StopRule r;
        r.kind = Kind::ResidualStagnation;
        r.stagnation_window = window;
        r.stagnation_improvement = improvement;
        return r;
    }
};

struct ProbeOptions {
    int cadence = 1;
    const DenseVector* x_star = nullptr;
    bool enabled = true;
};

struct IterationRecord {
    int k = 0;
    std::optional<double> rel_err_a_norm, true_res_norm, upd_res_norm, residual_gap_norm, nu_gap,
        w_gap_norm, s_gap_norm, lanczos_res_norm, succ_orth, alpha, beta, nu, nu_prime;
};

struct Summary {
    std::optional<int> iters_to_1e5;
    double min_log10_err = 0.0;
};

struct ConvergenceHistory {
    std::string problem_id;
    VariantConfig config;
    Preconditioner::Kind precond = Preconditioner::Kind::Identity;
    std::vector<IterationRecord> records;
    SolveStatus final_status;
    std::optional<Summary> summary;
};

inline ConvergenceHistory run(const VariantConfig& config, const SparseMatrix& a,
                              const Preconditioner& m, const DenseVector& b, const DenseVector& x0,
                              int max_iter, const StopRule& stop, const ProbeOptions& probe_opts) {
    if (max_iter < 0) throw std::invalid_argument("max_iter must be >= 0");
    config.validate();
    const auto n = static_cast<std::size_t>(a.n);
    if (b.size() != n || x0.size() != n)
        throw std::invalid_argument("right-hand side or initial guess dimension mismatch");
    if (probe_opts.x_star && probe_opts.x_star->size() != n)
        throw std::invalid_argument("x* dimension mismatch");
    const int precond = m.device_kind_for(a);
    const cgvk_variant_config c = config.to_c();
    const cgvk_stop_rule sr{static_cast<int>(stop.kind), stop.fixed_count, stop.error_threshold,
                            stop.stagnation_window, stop.stagnation_improvement};
    const cgvk_probe_options po{probe_opts.enabled ? 1 : 0, probe_opts.cadence,
                                probe_opts.x_star ? probe_opts.x_star->data() : nullptr};
    std::vector<cgvk_record> recs(static_cast<std::size_t>(max_iter) + 2);
    int nrec = 0;
    cgvk_solve_status fs{};
    cgvk_summary sm{};
    detail::check(cgvk_run(a.on_device(), &c, precond, b.data(), x0.data(), max_iter, &sr, &po, recs.data(), static_cast<int>(recs.size()),
                           &nrec, &fs, &sm, nullptr));
    ConvergenceHistory h;
    h.config = config;
    h.precond = m.kind;
    for (int q = 0; q < std::min(nrec, static_cast<int>(recs.size())); ++q) {
        const cgvk_record& r = recs[q];
        IterationRecord rec;
        rec.k = r.k;
        std::optional<double>* f[CGVK_REC_FIELDS] = {
            &rec.rel_err_a_norm, &rec.true_res_norm, &rec.upd_res_norm, &rec.residual_gap_norm,
            &rec.nu_gap, &rec.w_gap_norm, &rec.s_gap_norm, &rec.lanczos_res_norm, &rec.succ_orth,
            &rec.alpha, &rec.beta, &rec.nu, &rec.nu_prime};
        for (int i = 0; i < CGVK_REC_FIELDS; ++i)
            if (r.mask >> i & 1u) *f[i] = r.v[i];
        h.records.push_back(rec);
    }
    h.final_status.state = static_cast<SolveStatus::State>(fs.state);
    h.final_status.breakdown = static_cast<BreakdownReason>(fs.breakdown);
    h.final_status.criterion = static_cast<ConvergedBy>(fs.criterion);
    if (sm.has) {
        Summary s;
        if (sm.iters_to_1e5 >= 0) s.iters_to_1e5 = sm.iters_to_1e5;
        s.min_log10_err = sm.min_log10_err;
        h.summary = s;
    }
    return h;
}

}  // namespace cgv
