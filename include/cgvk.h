/* cgvk — B200-native preconditioned CG variants (arXiv 1905.01549), C ABI.
 *
 * This is the drop-in boundary for the reference's hot path. The reference
 * (/root/reference/proj) is a C++20 static library with no FFI; each entry
 * point below replaces one reference interface (file:line cited), with plain
 * pointers and sizes, host buffers in and out, and status codes that map 1:1
 * onto the reference's exception types:
 *
 *   CGVK_EINVAL  <-> std::invalid_argument  (dimension / config / CSR errors)
 *   CGVK_ESTATE  <-> std::logic_error       ("step() on a terminated solver")
 *   CGVK_ECUDA / CGVK_ENCCL / CGVK_ENOMEM   <-> std::runtime_error
 *
 * Numerical breakdown is NOT an error: it is reported through
 * cgvk_solver_status(), exactly as SolveStatus (inc/variants.hpp:62-86).
 * The C++ shim paper_1905_01549_b200/cpp/cgvariants/*.hpp rethrows these codes
 * so that cgv:: callers see the reference semantics.
 *
 * Threading: a matrix handle is immutable after creation and may be shared by
 * solvers on the same device (the reference borrows A read-only,
 * inc/variants.hpp:103-104): as there, a matrix must outlive the solvers
 * that use it. A solver handle is single-owner (inc/variants.hpp:95-97) and
 * owns its stream, graphs and device buffers. A communicator (row-partitioned
 * solves) is kept alive by the groups made over it, so it may be destroyed
 * before them.
 */
#ifndef CGVK_H
#define CGVK_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CGVK_VERSION 1

enum {
    CGVK_OK = 0,
    CGVK_EINVAL = -1,
    CGVK_ESTATE = -2,
    CGVK_ECUDA = -3,
    CGVK_ENCCL = -4,
    CGVK_ENOMEM = -5,
};

/* inc/variants.hpp:17-25 (same order) */
enum {
    CGVK_HS = 0,
    CGVK_CG_CG = 1,
    CGVK_M = 2,
    CGVK_PR = 3,
    CGVK_GV = 4,
    CGVK_PIPE_PR_M = 5,
    CGVK_PIPE_PR = 6,
};

/* inc/variants.hpp:28-32 (same order) */
enum { CGVK_NU_EXPANDED = 0, CGVK_NU_SIMPLIFIED = 1, CGVK_NU_MEURANT = 2 };

/* inc/preconditioner.hpp:13-14 */
enum { CGVK_PRECOND_IDENTITY = 0, CGVK_PRECOND_JACOBI = 1 };

/* SolveStatus::State, BreakdownReason, ConvergedBy (inc/variants.hpp:62-86).
 * CGVK_CONVERGED_BY_TOLERANCE is the relative-residual stop rule applied by
 * cgvk_solver_set_tolerance (the reference applies it in its harness, after
 * step()). */
enum { CGVK_RUNNING = 0, CGVK_BREAKDOWN = 1, CGVK_MAX_ITERATIONS = 2, CGVK_CONVERGED = 3 };
enum {
    CGVK_BREAKDOWN_NONE = 0,
    CGVK_BREAKDOWN_NU_PRIME_NONPOSITIVE = 1,
    CGVK_BREAKDOWN_NU_NONPOSITIVE = 2,
    CGVK_BREAKDOWN_MU_NONPOSITIVE = 3,
    CGVK_BREAKDOWN_NON_FINITE = 4,
};
enum {
    CGVK_CONVERGED_BY_ZERO_RESIDUAL = 0,
    CGVK_CONVERGED_BY_ERROR_THRESHOLD = 1,
    CGVK_CONVERGED_BY_STAGNATION = 2,
    CGVK_CONVERGED_BY_TOLERANCE = 3,
};

/* Working-vector ids for cgvk_solver_get_vector (SolverState fields,
 * inc/variants.hpp:108-111). */
enum {
    CGVK_VEC_X = 0, CGVK_VEC_R, CGVK_VEC_P, CGVK_VEC_S, CGVK_VEC_W, CGVK_VEC_U, CGVK_VEC_T,
    CGVK_VEC_R_TILDE, CGVK_VEC_S_TILDE, CGVK_VEC_W_TILDE, CGVK_VEC_U_TILDE,
};

/* Matrix creation flags. */
enum {
    CGVK_MATRIX_CHECK_SYMMETRIC = 1, /* is_symmetric (src/sparse_matrix.cpp:84-107) */
    CGVK_MATRIX_ENGINE_CSR = 2,      /* SpMV kernels: TMA-staged CSR tiles only */
    CGVK_MATRIX_ENGINE_BAND = 4,     /* SpMV kernels: band engine whenever it applies */
};

/* SpMV engine of a matrix (cgvk_matrix_engine). Without an ENGINE flag the
 * band engine (SELL-C-sigma + shared-memory x window) is chosen when every
 * tile's columns lie within a narrow band and rows are long; otherwise CSR
 * with x gathered through L1/L2. */
enum { CGVK_ENGINE_CSR = 0, CGVK_ENGINE_BAND = 1 };

/* POD mirror of VariantConfig (inc/variants.hpp:34-57). */
typedef struct cgvk_variant_config {
    int variant;
    int nu_expression;
    int recompute_nu;
    int recompute_w;
    int unsimplified_mu;
    int track_delta;
} cgvk_variant_config;

typedef struct cgvk_solve_status {
    int state;     /* CGVK_RUNNING ... */
    int breakdown; /* CGVK_BREAKDOWN_* */
    int criterion; /* CGVK_CONVERGED_BY_* */
    int k;         /* SolverState::k */
    int allocated_vectors; /* SolverState::allocated_vectors() */
} cgvk_solve_status;

/* SolverState scalars (inc/variants.hpp:122-130) plus the last <r,r>. */
typedef struct cgvk_scalars {
    double alpha, beta, nu, nu_prime, mu, delta, delta_hat, gamma, eta;
    double rr;
} cgvk_scalars;

/* SolverStats (inc/variants.hpp:88-93). */
typedef struct cgvk_stats {
    uint64_t spmv_calls, block_spmv_calls, precond_applies, reductions;
} cgvk_stats;

typedef struct cgvk_matrix_s* cgvk_matrix;
typedef struct cgvk_solver_s* cgvk_solver;

/* Thread-local message for the last non-OK return on this thread. */
const char* cgvk_last_error(void);
int cgvk_device_count(int* count);

/* VariantConfig::make / validate (src/variants.cpp:10-47). */
cgvk_variant_config cgvk_variant_config_make(int variant);
int cgvk_variant_config_validate(const cgvk_variant_config* cfg);

/* SparseMatrix upload (inc/sparse_matrix.hpp:16-23) with validate_csr
 * (src/sparse_matrix.cpp:64-82) run on the device; CGVK_EINVAL on any
 * violated invariant. Host arrays are the reference's int64/fp64 layout and
 * may be pageable or pinned. Device layout: int32 row_ptr/col_idx + fp64
 * values (12 B/nnz), requires nnz < 2^31. */
int cgvk_matrix_create_csr(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                           const double* values, int device, int flags, cgvk_matrix* out);
int cgvk_matrix_destroy(cgvk_matrix a);
int cgvk_matrix_info(cgvk_matrix a, int64_t* n, int64_t* nnz, int* device);
/* Engine the variant SpMV kernels use for `a` and, for the band engine, the
 * x-window half-width in 256-row tiles (0 for CSR). */
int cgvk_matrix_engine(cgvk_matrix a, int* engine, int* band_tiles);

/* spmv (inc/sparse_matrix.hpp:41-42, src/sparse_matrix.cpp:109-118): y = A*x,
 * per-row left-to-right, no FMA — bit-identical to the reference. */
int cgvk_spmv(cgvk_matrix a, const double* x, double* y);
/* block_spmv (inc/sparse_matrix.hpp:46-47, src/sparse_matrix.cpp:126-143). */
int cgvk_block_spmv(cgvk_matrix a, const double* x1, const double* x2, double* y1,
                    double* y2);
/* Preconditioner::jacobi (src/preconditioner.cpp:12-31): inv_diag = 1/a_ii;
 * CGVK_EINVAL when a diagonal entry is missing or <= 0. */
int cgvk_jacobi(cgvk_matrix a, double* inv_diag);
/* Preconditioner::apply (src/preconditioner.cpp:33-42). */
int cgvk_precond_apply(cgvk_matrix a, int kind, const double* in, double* out);
/* dot (inc/vector_ops.hpp:20-25) in the device's canonical reduction order
 * (reproduced bit-for-bit by oracle/cgv_oracle.c ORC_DOT_TREE). */
int cgvk_dot(cgvk_matrix a, const double* x, const double* y, double* out);
/* Device time (ms, mean of `reps` back-to-back launches, CUDA events) of the
 * L1 operators the reference's cost model abstracts (src/cost_model.cpp:15-30):
 * ms[CGVK_TIME_SPMV] y = A x, [CGVK_TIME_BLOCK_SPMV] (A x1, A x2) in one pass,
 * [CGVK_TIME_DOT] one global reduction (dot + last-CTA fold), [CGVK_TIME_COPY]
 * one n-vector copy. For calibration only (scripts/cost_model.py). */
enum { CGVK_TIME_SPMV = 0, CGVK_TIME_BLOCK_SPMV, CGVK_TIME_DOT, CGVK_TIME_COPY, CGVK_TIMED_OPS };
int cgvk_time_ops(cgvk_matrix a, int reps, double* ms);
/* Experiments only: per-CTA phase timestamps (ns) of the last update / SpMV
 * kernel launches, [2][1024][8]; CGVK_EINVAL unless built with CGVK_TIMELINE. */
int cgvk_debug_timeline(unsigned long long* out);
/* The reduction-tree parameters the oracle needs: rows per tile (= threads
 * per CTA), the CTA cap G and the tile order (0 strided, 1 contiguous). */
int cgvk_reduction_config(cgvk_matrix a, int* block, int* gmax, int* order);

/* initialize() (inc/variants.hpp:149-150, src/variants.cpp:354-444). The
 * status may already be terminal (zero initial residual, nu0/mu0 <= 0).
 * Stream-ordered: b and x0 are copied and the reference's initialization
 * (vectors, reductions, scalar checks) is enqueued on the solver's stream
 * without a host wait; cgvk_solver_status / _sync observe the result. Host
 * buffers must stay unchanged until the next synchronising call on the
 * solver when they are pinned (cudaMemcpyAsync semantics); pageable buffers
 * are copied before the call returns. Uploads of successive creations on one
 * device are issued in creation order. */
int cgvk_solver_create(cgvk_matrix a, const cgvk_variant_config* cfg, int precond,
                       const double* b, const double* x0, cgvk_solver* out);
int cgvk_solver_destroy(cgvk_solver s);
/* Relative-residual stop: terminate with CGVK_CONVERGED_BY_TOLERANCE after the
 * first step whose sqrt(<r,r>) <= rel_tol*||b||. rel_tol <= 0 disables it. */
int cgvk_solver_set_tolerance(cgvk_solver s, double rel_tol);
/* Enqueue up to n_iters step() calls (inc/variants.hpp:153) on the solver's
 * stream as CUDA-graph replays; returns immediately. Iterations after a
 * terminal status are device-side no-ops. CGVK_ESTATE if the status last
 * observed by the host is already terminal. */
int cgvk_solver_step(cgvk_solver s, int n_iters);
/* Wait for enqueued work and refresh the host mirror of the status. */
int cgvk_solver_sync(cgvk_solver s);
int cgvk_solver_status(cgvk_solver s, cgvk_solve_status* st, cgvk_scalars* sc,
                       cgvk_stats* stats);
/* Copy a working vector to the host in the reference's state (tilde vectors
 * that the fused schedule recomputes on the fly are materialised);
 * CGVK_EINVAL when the variant does not allocate it. Synchronises. */
int cgvk_solver_get_vector(cgvk_solver s, int which, double* out);
/* Enqueue the download of x (CGVK_VEC_X only; x_k is complete after every
 * step) on the solver's stream without waiting: `out` (preferably pinned,
 * cgvk_host_register) is valid after cgvk_solver_sync. */
int cgvk_solver_get_vector_async(cgvk_solver s, int which, double* out);
/* Stream order between two solvers on one device (an extension; the reference
 * runs solves one after another by construction): work enqueued on `s` from
 * now on starts after everything already enqueued on `prev` (upload, steps,
 * downloads), so a batch of solves can keep its copies overlapped while its
 * iterations do not interleave on the SMs. */
int cgvk_solver_after(cgvk_solver s, cgvk_solver prev);
/* ||b - A x_k|| with a fresh device spmv (diagnostics.cpp:19-24). */
int cgvk_solver_true_residual(cgvk_solver s, double* out);
/* sqrt(<r_j,r_j>) for j = 0..k as recorded on the device each iteration.
 * The device records the first CGVK_HISTORY_CAP entries (j < 131072); *len =
 * min(k + 1, CGVK_HISTORY_CAP), so a longer solve is visible to the caller as
 * *len < k + 1 (the Python and C++ mirrors raise on it). */
#define CGVK_HISTORY_CAP (1 << 17)
int cgvk_solver_history(cgvk_solver s, double* out, int cap, int* len);
/* The stream the solver enqueues on (cudaStream_t), for event timing. */
void* cgvk_solver_stream(cgvk_solver s);
/* Number of kernel launches one iteration makes (graph nodes / iteration):
 * 2, or 1 for PR / M, CG-CG, GV and pipe-PR on single-GPU problems that fit L2 (the
 * one-kernel schedule, same bits; environment CGVK_FUSE=0 turns it off). */
int cgvk_solver_launches_per_iter(cgvk_solver s);
/* Kernel launches of one cgvk_solver_step(s, n_iters) call on this rank: the
 * limit-setting kernel, the captured kernels of every replayed graph and the
 * plain launches of the remainder (including the closing tail kernel of each
 * chained run); NCCL's own kernels not counted. */
long long cgvk_solver_launches(cgvk_solver s, int n_iters);
/* Device-timed step(): CUDA events on the solver's stream around the enqueue
 * of n_iters graph-replayed iterations; synchronises. *iters = iterations
 * actually executed (fewer if the solver terminated). */
int cgvk_solver_time_steps(cgvk_solver s, int n_iters, double* ms, int* iters);
/* Per-kernel device times: n_iters iterations launched kernel by kernel (no
 * graph) with CUDA events around each launch on the solver's stream; returns
 * the summed milliseconds of the first (update) and second (SpMV) kernel. */
int cgvk_solver_profile(cgvk_solver s, int n_iters, double* k1_ms, double* k2_ms, int* iters);

/* run() (inc/runner.hpp:47-49) with StopRule::fixed(max_iter) and probes
 * off, plus an optional relative-residual tolerance: initialize, step until
 * terminal or max_iter, copy x back. Fills status/scalars when non-NULL. */
int cgvk_solve(cgvk_matrix a, const cgvk_variant_config* cfg, int precond, const double* b,
               const double* x0, int max_iter, double rel_tol, double* x_out,
               cgvk_solve_status* st, cgvk_scalars* sc);

/* ------------------------------------------------------ run() with probes
 * run() (inc/runner.hpp:47-49, src/runner.cpp:32-147) with its StopRule
 * (runner.hpp:9-36) and ProbeOptions (runner.hpp:38-42); every probe
 * quantity (src/diagnostics.cpp:11-72) and the three-term Lanczos residual
 * (:74-109) computed on the device from fresh products. */
enum { CGVK_STOP_FIXED = 0, CGVK_STOP_ERROR_REDUCTION = 1, CGVK_STOP_STAGNATION = 2 };
typedef struct cgvk_stop_rule {
    int kind;                      /* CGVK_STOP_* (reference default: stagnation) */
    int fixed_count;               /* StopRule::fixed */
    double error_threshold;        /* on ||e_k||_A/||e_0||_A, needs x* (1e-5) */
    int stagnation_window;         /* 50 */
    double stagnation_improvement; /* 0.01 */
} cgvk_stop_rule;
typedef struct cgvk_probe_options {
    int enabled;          /* reference default: 1 */
    int cadence;          /* record every m-th iteration (+ k = 0, terminal, stop) */
    const double* x_star; /* host, n; NULL disables rel_err_a_norm */
} cgvk_probe_options;
/* IterationRecord (inc/diagnostics.hpp:16-29): field f present iff mask bit f. */
enum {
    CGVK_REC_REL_ERR_A_NORM = 0, CGVK_REC_TRUE_RES_NORM, CGVK_REC_UPD_RES_NORM,
    CGVK_REC_RESIDUAL_GAP_NORM, CGVK_REC_NU_GAP, CGVK_REC_W_GAP_NORM, CGVK_REC_S_GAP_NORM,
    CGVK_REC_LANCZOS_RES_NORM, CGVK_REC_SUCC_ORTH, CGVK_REC_ALPHA, CGVK_REC_BETA, CGVK_REC_NU,
    CGVK_REC_NU_PRIME, CGVK_REC_FIELDS
};
typedef struct cgvk_record {
    int k;
    unsigned mask;
    double v[CGVK_REC_FIELDS];
} cgvk_record;
/* Summary (inc/diagnostics.hpp:54-57); has = 0 when absent. */
typedef struct cgvk_summary {
    int has;
    int iters_to_1e5; /* -1 when never reached */
    double min_log10_err;
} cgvk_summary;
/* Records beyond rec_cap are counted in *n_records but not stored. Errors as
 * the reference: max_iter < 0, error-reduction stop without x*, x0 == x*. */
int cgvk_run(cgvk_matrix a, const cgvk_variant_config* cfg, int precond, const double* b,
             const double* x0, int max_iter, const cgvk_stop_rule* stop,
             const cgvk_probe_options* probe, cgvk_record* records, int rec_cap, int* n_records,
             cgvk_solve_status* final_status, cgvk_summary* summary, double* x_out);

/* ---------------------------------------------------- row-partitioned solve
 * (SURVEY §8(e)); the reference has no distributed code. Rank r owns rows
 * [lo[r], lo[r+1]); SpMV rows stay bit-identical to the reference for any P,
 * dots are rank-local canonical trees summed in rank order. */
typedef struct cgvk_comm_s* cgvk_comm;

/* Contiguous row blocks cut at multiples of `align` (rows per plane: z-slabs). */
int cgvk_partition_rows(int64_t n, int nparts, int64_t align, int64_t* lo);
/* Halo plan of `rank` from its own rows (local row_ptr, global columns):
 * sizes4 = {lower halo, upper halo, rows sent down, rows sent up}; arrays
 * (nullable) receive the sorted global halo columns and local send rows. */
int cgvk_halo_plan(int64_t n, int nranks, const int64_t* lo, int rank, const int64_t* row_ptr,
                   const int64_t* col_idx, int64_t* sizes4, int64_t* lower, int64_t* upper,
                   int64_t* send_lo, int64_t* send_hi);
/* Rank-local column numbering of `rank`'s rows (global columns in col_idx,
 * local row_ptr from 0): own columns first, then the lower and upper halo
 * from *hbase = own rows rounded up to 32 (0 halo: *hbase = own rows).
 * Host only; cgvk_matrix_create_rank uses exactly this numbering. */
int cgvk_rank_local_columns(int64_t n, int nranks, const int64_t* lo, int rank, const int64_t* row_ptr,
                            const int64_t* col_idx, int64_t* local_col_idx, int64_t* hbase);
/* Rank-local matrix: rows [lo[rank], lo[rank+1]) in local numbering
 * [own | pad | lower halo | upper halo] (cgvk_rank_local_columns). */
int cgvk_matrix_create_rank(int64_t n, int nranks, int rank, const int64_t* lo, const int64_t* row_ptr,
                            const int64_t* col_idx, const double* values, int device, cgvk_matrix* out);
/* NCCL transport (one process per GPU; libnccl.so.2 is dlopen'ed). */
int cgvk_comm_nccl_unique_id(void* id128);
int cgvk_comm_create_nccl(const void* id128, int nranks, int rank, int device, cgvk_comm* out);
/* In-process transport: all ranks in this process on one device. */
int cgvk_comm_create_local(int nranks, int device, cgvk_comm* out);
int cgvk_comm_destroy(cgvk_comm c);
/* initialize() across the ranks this process drives (all of them for a local
 * comm, its own for NCCL); b/x0 are the local rows. */
int cgvk_group_create(cgvk_comm comm, int nlocal, const cgvk_matrix* As, const cgvk_variant_config* cfg,
                      int precond, const double* const* b, const double* const* x0, cgvk_solver* out);
/* Group flags. CGVK_GROUP_P2P: the iteration exchanges halos and rank totals
 * through peer memory inside the kernels (stores + stamps over NVLink, no
 * NCCL call and no exchange launch per iteration; GV / pipe-PR fold their
 * K1 reduction in the next K1, so it overlaps the SpMV). Needs z-slab-like
 * ranks (send rows = a prefix and a suffix of the rank's rows), the CSR
 * engine and <= 8 ranks; NCCL groups exchange CUDA IPC handles once.
 * Bit-identical to the default transport. */
enum { CGVK_GROUP_P2P = 1 };
int cgvk_group_create_ex(cgvk_comm comm, int nlocal, const cgvk_matrix* As, const cgvk_variant_config* cfg,
                         int precond, const double* const* b, const double* const* x0, int flags,
                         cgvk_solver* out);
/* CGVK_GROUP_P2P or 0 for a group member; -1 otherwise. */
int cgvk_group_transport(cgvk_solver s);
/* n_iters step() calls on every local rank (graph replays incl. exchanges). */
int cgvk_group_step(const cgvk_solver* solvers, int nlocal, int n_iters);
/* ||b - A x|| over all ranks. */
int cgvk_group_true_residual(const cgvk_solver* solvers, int nlocal, double* out);

/* Page-lock / unlock a host buffer (cudaHostRegister) for the e2e path. */
int cgvk_host_register(void* ptr, uint64_t bytes);
int cgvk_host_unregister(void* ptr);

#ifdef __cplusplus
}
#endif
#endif /* CGVK_H */
