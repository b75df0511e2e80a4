/* TEST INFRASTRUCTURE ONLY — the CPU oracle for the PCG-variant hot path.
 *
 * A plain-C restatement of the reference algorithm (proj/src/variants.cpp,
 * sparse_matrix.cpp, preconditioner.cpp, inc/vector_ops.hpp), used by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg only — never by the
 * product library. Parity of this restatement is pinned against the
 * reference itself (oracle/_ref/libcgvref.so, bitwise in ORC_DOT_SEQ mode) and
 * against the paper's Table-3 counts (tests/test_oracle.py).
 *
 * Dot-product order is selectable:
 *   ORC_DOT_SEQ   left-to-right, exactly inc/vector_ops.hpp:20-25 (the reference)
 *   ORC_DOT_TREE  the GPU's canonical reduction tree: tiles of
 *                 `block` rows, one row per thread; thread t of CTA b sums its
 *                 rows of the contiguous tiles [b*T/G, (b+1)*T/G) (T tiles,
 *                 G = min(gmax, T)) sequentially; a warp
 *                 shfl_down tree (16,8,4,2,1) and a cross-warp tree give the
 *                 CTA partial; the last CTA sums partials j = t mod block
 *                 sequentially per thread and applies the same block tree.
 *                 With it the GPU path must match bit-for-bit.
 *   ORC_DOT_PART  ORC_DOT_TREE on each row block of a partition, the block
 *                 partials summed in rank order (the multi-GPU order).
 */
#ifndef CGV_ORACLE_H
#define CGV_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_DOT_SEQ = 0, ORC_DOT_TREE = 1, ORC_DOT_PART = 2 };

typedef struct orc_dotcfg {
    int mode;
    int block;             /* rows per tile = threads per CTA (multiple of 32, pow2) */
    int gmax;              /* CTA count cap; G = min(gmax, ntiles) */
    int nparts;            /* ORC_DOT_PART only */
    const int64_t* part_lo; /* nparts+1 row offsets */
    int order;             /* tile order: 0 strided (b, b+G, ...), 1 contiguous blocks */
} orc_dotcfg;

typedef struct orc_solver orc_solver;

double orc_dot(int64_t n, const double* x, const double* y, const orc_dotcfg* cfg);
void orc_spmv(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
              const double* x, double* y);
void orc_block_spmv(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                    const double* x1, const double* x2, double* y1, double* y2);
/* 0 ok, -1 missing or non-positive diagonal (preconditioner.cpp:12-31) */
int orc_jacobi(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
               double* inv_diag);
/* 0 ok, -1 invalid (sparse_matrix.cpp:64-82) */
int orc_validate_csr(int64_t n, const int64_t* rp, const int64_t* ci, int64_t nnz);

/* Returns NULL with *err = -1 (invalid_argument) on a bad config or a
 * Jacobi failure. The CSR arrays and b are borrowed, not copied. */
orc_solver* orc_solver_create(int64_t n, const int64_t* rp, const int64_t* ci,
                              const double* v, int variant, int nu_expr, int recompute_nu,
                              int recompute_w, int unsimplified_mu, int track_delta,
                              int precond, const double* b, const double* x0,
                              const orc_dotcfg* dcfg, int* err);
void orc_solver_destroy(orc_solver* s);
/* 0 ok, -2 step() on a terminated solver (variants.cpp:447) */
int orc_solver_step(orc_solver* s);
void orc_solver_state(const orc_solver* s, int* k, int* status4, double* scalars9,
                      uint64_t* stats4);
int orc_solver_vector(const orc_solver* s, int which, double* out);
int orc_solve(orc_solver* s, const double* b, int max_iter, double tol, double* upd_hist,
              double* true_hist, int true_cap);
double orc_time_steps(orc_solver* s, int iters, int* taken);
int orc_anorm_run(orc_solver* s, const double* x_star, int max_iter, double threshold,
                  int* iters_to_1e5, double* min_log10_err, int* final_state);
int orc_config_validate(int variant, int nu_expr, int recompute_nu, int recompute_w,
                        int unsimplified_mu, int track_delta);

#ifdef __cplusplus
}
#endif
#endif
