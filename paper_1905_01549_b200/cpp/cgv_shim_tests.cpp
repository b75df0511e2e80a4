// Reference-style tests through the cgv:: shim (the reference's own API over
// the B200 path). Mirrors proj/tests/test_variants.cpp, test_sparse_matrix.cpp
// and test_preconditioner.cpp; run on a GPU box by tests/test_cpp_shim.py.
#include "cgvariants/preconditioner.hpp"
#include "cgvariants/runner.hpp"
#include "cgvariants/sparse_matrix.hpp"
#include "cgvariants/variants.hpp"
#include "cgvariants/vector_ops.hpp"

#include <cstdio>
#include <cstring>
#include <functional>
#include <random>
#include <thread>

using namespace cgv;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                                  \
    do {                                                                             \
        ++g_checks;                                                                  \
        if (!(cond)) {                                                               \
            ++g_fail;                                                                \
            std::fprintf(stderr, "%s:%d: CHECK failed: %s\n", __FILE__, __LINE__, #cond); \
        }                                                                            \
    } while (0)
#define CHECK_THROWS_AS(expr, T)          \
    do {                                  \
        bool thrown_ = false;             \
        try {                             \
            expr;                         \
        } catch (const T&) {              \
            thrown_ = true;               \
        }                                 \
        CHECK(thrown_);                   \
    } while (0)

static SparseMatrix identity_matrix(Index n) {
    std::vector<Triplet> t;
    for (Index i = 0; i < n; ++i) t.emplace_back(i, i, 1.0);
    return csr_from_triplets(n, std::move(t));
}

static DenseVector random_vector(Index n, std::uint64_t seed) {
    std::mt19937_64 eng(seed);
    std::uniform_real_distribution<double> dist(-1.0, 1.0);
    DenseVector x(static_cast<std::size_t>(n));
    for (auto& v : x) v = dist(eng);
    return x;
}

static SparseMatrix laplace2d(Index N) {
    std::vector<Triplet> t;
    for (Index y = 0; y < N; ++y)
        for (Index x = 0; x < N; ++x) {
            const Index i = x + N * y;
            t.emplace_back(i, i, 4.0);
            if (x > 0) t.emplace_back(i, i - 1, -1.0);
            if (x < N - 1) t.emplace_back(i, i + 1, -1.0);
            if (y > 0) t.emplace_back(i, i - N, -1.0);
            if (y < N - 1) t.emplace_back(i, i + N, -1.0);
        }
    return csr_from_triplets(N * N, std::move(t));
}

static const Variant kAll[] = {Variant::HS, Variant::CG_CG, Variant::M, Variant::PR,
                               Variant::GV, Variant::PIPE_PR_M, Variant::PIPE_PR};

static void test_initialize_identity() {  // test_variants.cpp:37-49
    const SparseMatrix a = identity_matrix(8);
    const Preconditioner m = Preconditioner::identity();
    const DenseVector b = random_vector(8, 1), x0(8, 0.0);
    for (Variant v : kAll) {
        SolverState st = initialize(VariantConfig::make(v), a, m, b, x0);
        CHECK(st.status.running());
        CHECK(st.p == b);
        CHECK(st.s == b);
        CHECK(st.alpha == 1.0);
    }
}

static void test_one_step_identity() {  // test_variants.cpp:74-89
    const SparseMatrix a = identity_matrix(10);
    const Preconditioner m = Preconditioner::identity();
    const DenseVector b = random_vector(10, 2), x0(10, 0.0);
    for (Variant v : kAll) {
        SolverState st = initialize(VariantConfig::make(v), a, m, b, x0);
        step(st);
        CHECK(st.k == 1);
        CHECK(st.x == b);
        CHECK(norm2(st.r) == 0.0);
        CHECK(st.status.state == SolveStatus::State::Converged);
        CHECK_THROWS_AS(step(st), std::logic_error);
    }
}

static void test_cg_cg_equals_hs() {  // test_variants.cpp:113-125
    const SparseMatrix a = identity_matrix(12);
    const Preconditioner m = Preconditioner::identity();
    const DenseVector b = random_vector(12, 5), x0(12, 0.0);
    SolverState hs = initialize(VariantConfig::make(Variant::HS), a, m, b, x0);
    SolverState cg = initialize(VariantConfig::make(Variant::CG_CG), a, m, b, x0);
    step(hs);
    step(cg);
    CHECK(hs.x == cg.x);
    CHECK(hs.r == cg.r);
}

static void test_allocations_and_counters() {  // test_variants.cpp:194-263
    const SparseMatrix a = laplace2d(12);
    const DenseVector b = random_vector(a.n, 6), x0(a.n, 0.0);
    const Preconditioner none = Preconditioner::identity();
    const Preconditioner jac = Preconditioner::jacobi(a);
    const int plain[] = {4, 5, 4, 4, 7, 6, 6}, prec[] = {5, 6, 6, 6, 10, 10, 10};
    const unsigned scal[] = {2, 2, 3, 4, 2, 3, 4};
    for (int i = 0; i < 7; ++i) {
        SolverState p0 = initialize(VariantConfig::make(kAll[i]), a, none, b, x0);
        SolverState p1 = initialize(VariantConfig::make(kAll[i]), a, jac, b, x0);
        CHECK(p0.allocated_vectors() == plain[i]);
        CHECK(p1.allocated_vectors() == prec[i]);
        const auto base = p0.stats;
        step(p0);
        CHECK(p0.stats.reductions - base.reductions == scal[i]);
        const bool pipe = kAll[i] == Variant::PIPE_PR || kAll[i] == Variant::PIPE_PR_M;
        CHECK(p0.stats.block_spmv_calls - base.block_spmv_calls == (pipe ? 1u : 0u));
        CHECK(p0.stats.spmv_calls - base.spmv_calls == (pipe ? 0u : 1u));
    }
}

static void test_block_spmv_and_jacobi() {  // test_sparse_matrix.cpp:56-78, test_preconditioner.cpp
    const SparseMatrix a = laplace2d(9);
    const DenseVector x1 = random_vector(a.n, 3), x2 = random_vector(a.n, 4);
    DenseVector y1(a.n), y2(a.n);
    block_spmv(a, x1, x2, y1, y2);
    CHECK(y1 == spmv(a, x1));
    CHECK(y2 == spmv(a, x2));
    CHECK(spmv(identity_matrix(17), random_vector(17, 1)) == random_vector(17, 1));
    DenseVector bad(3, 1.0), out(a.n);
    CHECK_THROWS_AS(spmv(a, bad, out), std::invalid_argument);
    const SparseMatrix two = csr_from_triplets(2, {{0, 0, 2.0}, {0, 1, 1.0}, {1, 0, 1.0}, {1, 1, 4.0}});
    const Preconditioner m = Preconditioner::jacobi(two);
    CHECK(m.inv_diag[0] == 0.5 && m.inv_diag[1] == 0.25);
    const SparseMatrix missing = csr_from_triplets(2, {{0, 1, 1.0}, {1, 0, 1.0}});
    CHECK_THROWS_AS(Preconditioner::jacobi(missing), std::invalid_argument);
    CHECK(is_symmetric(a));
    const SparseMatrix asym = csr_from_triplets(2, {{0, 0, 2.0}, {0, 1, 1.0}, {1, 0, 0.5}, {1, 1, 2.0}});
    CHECK(!is_symmetric(asym));
}

static void test_validate() {  // test_variants.cpp:301-317
    VariantConfig c = VariantConfig::make(Variant::HS);
    c.recompute_w = false;
    CHECK_THROWS_AS(c.validate(), std::invalid_argument);
    c = VariantConfig::make(Variant::PR);
    c.unsimplified_mu = true;
    CHECK_THROWS_AS(c.validate(), std::invalid_argument);
    c = VariantConfig::make(Variant::CG_CG);
    c.unsimplified_mu = true;
    c.validate();
}

static void test_run_fixed() {  // runner.hpp:47-49 with StopRule::fixed
    const SparseMatrix a = laplace2d(20);
    const Preconditioner m = Preconditioner::jacobi(a);
    const DenseVector xs = random_vector(a.n, 9);
    const DenseVector b = spmv(a, xs), x0(a.n, 0.0);
    for (Variant v : kAll) {
        ProbeOptions probe;
        probe.cadence = 10;
        const ConvergenceHistory h = run(VariantConfig::make(v), a, m, b, x0, 50, StopRule::fixed(50), probe);
        CHECK(h.final_status.state == SolveStatus::State::MaxIterations);
        CHECK(h.records.size() == 6);
        CHECK(h.records.back().k == 50);
        CHECK(*h.records.back().upd_res_norm < 1e-3 * *h.records.front().upd_res_norm);
        CHECK(*h.records.back().true_res_norm < 1e-3 * *h.records.front().true_res_norm);
        SolverState st = initialize(VariantConfig::make(v), a, m, b, x0);
        st.sync_host = false;
        step_n(st, 400, 1e-10);
        CHECK(st.status.state == SolveStatus::State::Converged);
        CHECK(st.status.criterion == ConvergedBy::Tolerance);
    }
}

static void test_run_probes() {  // runner.cpp:32-147 + diagnostics.cpp on the device
    const SparseMatrix a = laplace2d(20);
    const Preconditioner m = Preconditioner::jacobi(a);
    const DenseVector xs = random_vector(a.n, 11);
    const DenseVector b = spmv(a, xs), x0(a.n, 0.0);
    for (Variant v : kAll) {
        ProbeOptions probe;
        probe.x_star = &xs;
        const ConvergenceHistory h =
            run(VariantConfig::make(v), a, m, b, x0, 500, StopRule::error_reduction(1e-5), probe);
        CHECK(h.final_status.state == SolveStatus::State::Converged);
        CHECK(h.final_status.criterion == ConvergedBy::ErrorThreshold);
        CHECK(h.summary.has_value() && h.summary->iters_to_1e5.has_value());
        CHECK(*h.summary->iters_to_1e5 == h.records.back().k);
        CHECK(*h.records.front().rel_err_a_norm == 1.0);
        CHECK(*h.records.back().rel_err_a_norm < 1e-5);
        CHECK(h.records.size() >= 3 && h.records[2].lanczos_res_norm.has_value());
        CHECK(h.records[1].succ_orth.has_value() && std::abs(*h.records[1].succ_orth) < 1e-8);
        CHECK(*h.records.back().residual_gap_norm < 1e-8 * *h.records.front().true_res_norm);
        const bool pipelined = v == Variant::GV || v == Variant::PIPE_PR || v == Variant::PIPE_PR_M;
        CHECK(h.records.back().s_gap_norm.has_value() == pipelined);
        CHECK(h.records.back().w_gap_norm.has_value() == pipelined);
        const bool predictor = v == Variant::M || v == Variant::PR || v == Variant::PIPE_PR ||
                               v == Variant::PIPE_PR_M;
        CHECK(h.records.back().nu_gap.has_value() == predictor);
        // default rule: residual stagnation, probes on
        const ConvergenceHistory g = run(VariantConfig::make(v), a, m, b, x0, 2000, StopRule{}, ProbeOptions{});
        CHECK(g.final_status.state == SolveStatus::State::Converged);
        CHECK(g.final_status.criterion == ConvergedBy::Stagnation);
    }
    CHECK_THROWS_AS(run(VariantConfig::make(Variant::HS), a, m, b, x0, 5, StopRule::error_reduction(1e-5),
                        ProbeOptions{}),
                    std::invalid_argument);
}

// host-only: no device call (run on CPU by tests/test_cpp_shim.py --host)
static void test_csr_from_triplets() {  // sparse_matrix.hpp:25-27
    // unsorted input, a repeated position summed in input order, an exact-zero sum dropped
    const SparseMatrix a = csr_from_triplets(3, {{2, 1, 1.0}, {0, 2, 0.5}, {0, 0, 1e16}, {1, 1, 3.0},
                                                 {0, 0, 1.0}, {2, 0, 2.0}, {0, 0, -1e16}, {1, 0, 7.0},
                                                 {1, 0, -7.0}});
    // row 0: (1e16 + 1) + -1e16 == 0 -> dropped; row 1: 7 + -7 == 0 -> dropped
    CHECK((a.row_ptr == std::vector<Index>{0, 1, 2, 4}));
    CHECK((a.col_idx == std::vector<Index>{2, 1, 0, 1}));
    CHECK((a.values == std::vector<double>{0.5, 3.0, 2.0, 1.0}));
    // duplicates fold in input order, not sorted by value
    volatile double p1 = 0.1, p2 = 0.2, p3 = -0.3;
    const SparseMatrix c = csr_from_triplets(1, {{0, 0, 0.1}, {0, 0, 0.2}, {0, 0, -0.3}});
    const SparseMatrix d = csr_from_triplets(1, {{0, 0, -0.3}, {0, 0, 0.2}, {0, 0, 0.1}});
    CHECK(c.nnz() == 1 && c.values[0] == (p1 + p2) + p3);
    CHECK(d.nnz() == 1 && d.values[0] == (p3 + p2) + p1 && c.values[0] != d.values[0]);
    CHECK_THROWS_AS(csr_from_triplets(2, {{0, 2, 1.0}}), std::invalid_argument);
    CHECK_THROWS_AS(csr_from_triplets(2, {{-1, 0, 1.0}}), std::invalid_argument);
    const SparseMatrix e = csr_from_triplets(4, {});
    CHECK((e.row_ptr == std::vector<Index>{0, 0, 0, 0, 0}) && e.nnz() == 0);
    const DenseVector x{1.0, 2.0, 3.0}, y{4.0, 5.0, 6.0};
    CHECK(dot(x, y) == ((0.0 + 4.0) + 10.0) + 18.0);
    CHECK(norm2(x) == std::sqrt(14.0));
    CHECK_THROWS_AS(dot(x, DenseVector{1.0}), std::invalid_argument);
}

static void test_shared_matrix_threads() {  // experiment.cpp:317-322: one A, concurrent solves
    const SparseMatrix a = laplace2d(24);
    const Preconditioner m = Preconditioner::jacobi(a);
    const DenseVector b = spmv(a, random_vector(a.n, 5)), x0(a.n, 0.0);
    const SparseMatrix fresh{a.n, a.row_ptr, a.col_idx, a.values, {}};  // not yet uploaded
    std::vector<cgvk_matrix> handles(8);
    std::vector<std::thread> th;
    for (int i = 0; i < 8; ++i) th.emplace_back([&, i] { handles[i] = fresh.on_device(); });
    for (auto& t : th) t.join();
    for (int i = 1; i < 8; ++i) CHECK(handles[i] == handles[0]);  // one upload
    // a copy owns its own device matrix: editing it changes its products only
    SparseMatrix edited = a;
    for (double& v : edited.values) v *= 2.0;
    const DenseVector xa = random_vector(a.n, 6);
    const DenseVector ya = spmv(a, xa), ye = spmv(edited, xa);
    bool doubled = true;
    for (std::size_t i = 0; i < ya.size(); ++i) doubled = doubled && ye[i] == 2.0 * ya[i];
    CHECK(doubled);
    CHECK(edited.on_device() != a.on_device());
    // a Jacobi preconditioner is tied to its matrix and to its inv_diag as built
    CHECK_THROWS_AS(initialize(VariantConfig::make(Variant::HS), edited, m, b, x0), std::invalid_argument);
    Preconditioner tampered = m;
    tampered.inv_diag[3] *= 2.0;
    CHECK_THROWS_AS(initialize(VariantConfig::make(Variant::HS), a, tampered, b, x0), std::invalid_argument);
    CHECK_THROWS_AS(run(VariantConfig::make(Variant::PR), a, tampered, b, x0, 5, StopRule::fixed(5), ProbeOptions{}),
                    std::invalid_argument);
    SolverState st = initialize(VariantConfig::make(Variant::HS), a, m, b, x0);  // the untouched one is fine
    CHECK(st.status.running());
}

int main(int argc, char** argv) {
    if (argc > 1 && std::strcmp(argv[1], "--host") == 0) {
        test_csr_from_triplets();
        std::printf("[%s] csr_from_triplets\n%d checks, %d failures\n", g_fail ? "FAIL" : "ok", g_checks, g_fail);
        return g_fail ? 1 : 0;
    }
    const std::pair<const char*, std::function<void()>> tests[] = {
        {"csr_from_triplets", test_csr_from_triplets},
        {"shared_matrix_threads", test_shared_matrix_threads},
        {"initialize_identity", test_initialize_identity},
        {"one_step_identity", test_one_step_identity},
        {"cg_cg_equals_hs", test_cg_cg_equals_hs},
        {"allocations_and_counters", test_allocations_and_counters},
        {"block_spmv_and_jacobi", test_block_spmv_and_jacobi},
        {"validate", test_validate},
        {"run_fixed", test_run_fixed},
        {"run_probes", test_run_probes},
    };
    for (const auto& [name, fn] : tests) {
        const int before = g_fail;
        try {
            fn();
        } catch (const std::exception& e) {
            ++g_fail;
            std::fprintf(stderr, "%s: unexpected exception: %s\n", name, e.what());
        }
        std::printf("[%s] %s\n", g_fail == before ? "ok" : "FAIL", name);
    }
    std::printf("%d checks, %d failures\n", g_checks, g_fail);
    return g_fail ? 1 : 0;
}
