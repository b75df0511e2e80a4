/* Synthetic input generators. Host-only C. */
#ifndef CGVK_GEN_H
#define CGVK_GEN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* CSR in the reference's host layout (int64 indices, fp64 values,
 * proj/include/cgvariants/sparse_matrix.hpp:16-23). */
typedef struct cgvk_csr {
    int64_t n;
    int64_t nnz;
    int64_t* row_ptr;
    int64_t* col_idx;
    double* values;
} cgvk_csr;

void cgvk_csr_free(cgvk_csr* a);
void cgvk_gen_mt19937_64(uint64_t seed, int64_t count, uint64_t* out);
void cgvk_gen_xstar(int64_t n, uint64_t seed, double* out);
cgvk_csr* cgvk_gen_poisson(int dim, int64_t N);
cgvk_csr* cgvk_gen_varcoef(int64_t N, uint64_t seed, double sigma);
cgvk_csr* cgvk_gen_random_spd(int64_t n, int per_row, int64_t band, uint64_t seed);
void cgvk_gen_spmv(const cgvk_csr* a, const double* x, double* y);

#ifdef __cplusplus
}
#endif
#endif
