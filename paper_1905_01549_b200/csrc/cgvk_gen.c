/* Synthetic inputs for the BASELINE.json configs.
 *
 * Host-only, deterministic, and shared by the GPU path, the oracle harness and
 * bench.py so that every arm sees the same CSR arrays, x* and b. Matrices are
 * built directly in sorted CSR order (no triplet sort), with full symmetric
 * storage and bit-symmetric values (the invariant of
 * proj/include/cgvariants/sparse_matrix.hpp:11-15).
 *
 * RNG: std::mt19937_64 restated (checked against libstdc++ in
 * tests/test_generators.py), uniform u01 = ((e>>11)+0.5)*2^-53 and Box-Muller
 * with a cached spare, the recipe of proj/src/model_problem.cpp:15-42. */
#include "cgvk_gen.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------- mt19937_64 */

typedef struct {
    uint64_t mt[312];
    int mti;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->mti = 312;
}

static uint64_t mt64_next(mt64* g) {
    static const uint64_t mag01[2] = {0ULL, 0xB5026F5AA96619E9ULL};
    const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
    if (g->mti >= 312) {
        int i;
        uint64_t x;
        for (i = 0; i < 312 - 156; ++i) {
            x = (g->mt[i] & UM) | (g->mt[i + 1] & LM);
            g->mt[i] = g->mt[i + 156] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
        }
        for (; i < 311; ++i) {
            x = (g->mt[i] & UM) | (g->mt[i + 1] & LM);
            g->mt[i] = g->mt[i + (156 - 312)] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
        }
        x = (g->mt[311] & UM) | (g->mt[0] & LM);
        g->mt[311] = g->mt[155] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
        g->mti = 0;
    }
    uint64_t x = g->mt[g->mti++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
}

static double u01(mt64* g) { return ((double)(mt64_next(g) >> 11) + 0.5) * 0x1.0p-53; }

void cgvk_gen_mt19937_64(uint64_t seed, int64_t count, uint64_t* out) {
    mt64* g = (mt64*)malloc(sizeof(mt64));
    mt64_seed(g, seed);
    for (int64_t i = 0; i < count; ++i) out[i] = mt64_next(g);
    free(g);
}

/* x*_i = 2*u01 - 1 from its own engine (App. B) */
void cgvk_gen_xstar(int64_t n, uint64_t seed, double* out) {
    mt64* g = (mt64*)malloc(sizeof(mt64));
    mt64_seed(g, seed);
    for (int64_t i = 0; i < n; ++i) out[i] = 2.0 * u01(g) - 1.0;
    free(g);
}

/* ----------------------------------------------------------- helpers */

static cgvk_csr* csr_alloc(int64_t n, int64_t nnz) {
    cgvk_csr* a = (cgvk_csr*)calloc(1, sizeof(cgvk_csr));
    a->n = n;
    a->nnz = nnz;
    a->row_ptr = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
    a->col_idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nnz ? nnz : 1));
    a->values = (double*)malloc(sizeof(double) * (size_t)(nnz ? nnz : 1));
    return a;
}

void cgvk_csr_free(cgvk_csr* a) {
    if (!a) return;
    free(a->row_ptr);
    free(a->col_idx);
    free(a->values);
    free(a);
}

/* --------------------------------------------- Dirichlet Laplacians */

/* 5-point (dim=2) or 7-point (dim=3) Laplacian on an N^dim interior grid,
 * h^2 scaled out: diagonal 2*dim, -1 per in-grid neighbour, lexicographic
 * rows i = x + N*(y + N*z). nnz = 5n-4N (2D), 7n-6N^2 (3D). */
cgvk_csr* cgvk_gen_poisson(int dim, int64_t N) {
    if ((dim != 2 && dim != 3) || N < 1) return NULL;
    const int64_t n = dim == 2 ? N * N : N * N * N;
    const int64_t nnz = dim == 2 ? 5 * n - 4 * N : 7 * n - 6 * N * N;
    cgvk_csr* a = csr_alloc(n, nnz);
    const int64_t NN = N * N;
    int64_t k = 0;
    for (int64_t i = 0; i < n; ++i) {
        a->row_ptr[i] = k;
        const int64_t x = i % N, y = (i / N) % N, z = dim == 3 ? i / NN : 0;
#define PUT(c, v) (a->col_idx[k] = (c), a->values[k] = (v), ++k)
        if (dim == 3 && z > 0) PUT(i - NN, -1.0);
        if (y > 0) PUT(i - N, -1.0);
        if (x > 0) PUT(i - 1, -1.0);
        PUT(i, 2.0 * dim);
        if (x < N - 1) PUT(i + 1, -1.0);
        if (y < N - 1) PUT(i + N, -1.0);
        if (dim == 3 && z < N - 1) PUT(i + NN, -1.0);
#undef PUT
    }
    a->row_ptr[n] = k;
    return a;
}

/* ------------------------------------- variable-coefficient diffusion */

/* 7-point finite-volume diffusion on N^3 cells, k_c = exp(sigma*g_c) with g_c
 * i.i.d. N(0,1) (white-noise field, one Box-Muller draw per cell in row order
 * from mt19937_64(seed)); face coefficient = harmonic mean
 * 2*(k_a*k_b)/(k_a+k_b); boundary faces are Dirichlet at half-cell distance
 * (2*k_c on the diagonal); diagonal = sum of the six face terms in the order
 * -z,-y,-x,+x,+y,+z; off-diagonals = -face. */
cgvk_csr* cgvk_gen_varcoef(int64_t N, uint64_t seed, double sigma) {
    if (N < 1) return NULL;
    const int64_t n = N * N * N, NN = N * N;
    double* kc = (double*)malloc(sizeof(double) * (size_t)n);
    mt64* g = (mt64*)malloc(sizeof(mt64));
    mt64_seed(g, seed);
    int have_spare = 0;
    double spare = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        double gi;
        if (have_spare) {
            have_spare = 0;
            gi = spare;
        } else {
            const double u1 = u01(g), u2 = u01(g);
            const double radius = sqrt(-2.0 * log(u1));
            const double angle = 2.0 * M_PI * u2;
            spare = radius * sin(angle);
            have_spare = 1;
            gi = radius * cos(angle);
        }
        kc[i] = exp(sigma * gi);
    }
    free(g);
    const int64_t nnz = 7 * n - 6 * NN;
    cgvk_csr* a = csr_alloc(n, nnz);
    int64_t k = 0;
    for (int64_t i = 0; i < n; ++i) {
        const int64_t x = i % N, y = (i / N) % N, z = i / NN;
        const double ki = kc[i];
        /* neighbour offsets in the diagonal's summation order -z,-y,-x,+x,+y,+z */
        const int64_t off[6] = {-NN, -N, -1, 1, N, NN};
        const int inside[6] = {z > 0, y > 0, x > 0, x < N - 1, y < N - 1, z < N - 1};
        double face[6];
        double diag = 0.0;
        for (int d = 0; d < 6; ++d) {
            if (inside[d]) {
                const double kj = kc[i + off[d]];
                /* identical bits for (a,b) and (b,a): * and + commute exactly */
                face[d] = 2.0 * (ki * kj) / (ki + kj);
            } else {
                face[d] = 2.0 * ki;
            }
            diag += face[d];
        }
        a->row_ptr[i] = k;
        for (int d = 0; d < 3; ++d)
            if (inside[d]) {
                a->col_idx[k] = i + off[d];
                a->values[k++] = -face[d];
            }
        a->col_idx[k] = i;
        a->values[k++] = diag;
        for (int d = 3; d < 6; ++d)
            if (inside[d]) {
                a->col_idx[k] = i + off[d];
                a->values[k++] = -face[d];
            }
    }
    a->row_ptr[n] = k;
    free(kc);
    return a;
}

/* ------------------------------------------------- random banded SPD */

typedef struct {
    int64_t j;
    double v;
    int order;
} draw_t;

/* Per row i, `per_row` (offset, value) draws j = i+1+floor(u01*band),
 * v = -u01 (draws with j >= n are discarded after both numbers are drawn);
 * mirrored to (j,i); duplicates summed in draw order; diagonal = sum of
 * |off-diagonals| in increasing column order + 1e-3; then the symmetric
 * scaling a_ij*(s_i*s_j), s_i = 10^(6*u01-3), drawn after all rows. */
cgvk_csr* cgvk_gen_random_spd(int64_t n, int per_row, int64_t band, uint64_t seed) {
    if (n < 1 || per_row < 0 || per_row > 64 || band < 1) return NULL;
    mt64* g = (mt64*)malloc(sizeof(mt64));
    mt64_seed(g, seed);
    /* upper entries per row, deduplicated and sorted by column */
    int64_t* ucnt = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
    int64_t* uj = (int64_t*)malloc(sizeof(int64_t) * (size_t)n * (size_t)per_row);
    double* uv = (double*)malloc(sizeof(double) * (size_t)n * (size_t)per_row);
    int64_t* lcnt = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
    draw_t d[64];
    for (int64_t i = 0; i < n; ++i) {
        int m = 0;
        for (int t = 0; t < per_row; ++t) {
            const double uo = u01(g);
            const double uvv = u01(g);
            const int64_t j = i + 1 + (int64_t)floor(uo * (double)band);
            if (j >= n) continue;
            d[m].j = j;
            d[m].v = -uvv;
            d[m].order = t;
            ++m;
        }
        /* insertion sort by (j, draw order): stable */
        for (int a = 1; a < m; ++a) {
            draw_t key = d[a];
            int b = a - 1;
            while (b >= 0 && d[b].j > key.j) {
                d[b + 1] = d[b];
                --b;
            }
            d[b + 1] = key;
        }
        int64_t c = 0;
        int64_t* rowj = uj + i * per_row;
        double* rowv = uv + i * per_row;
        for (int a = 0; a < m;) {
            double sum = d[a].v;
            int b = a + 1;
            while (b < m && d[b].j == d[a].j) sum += d[b++].v;
            rowj[c] = d[a].j;
            rowv[c] = sum;
            ++c;
            lcnt[d[a].j]++;
            a = b;
        }
        ucnt[i] = c;
    }
    double* s = (double*)malloc(sizeof(double) * (size_t)n);
    for (int64_t i = 0; i < n; ++i) s[i] = pow(10.0, 6.0 * u01(g) - 3.0);
    free(g);

    int64_t nnz = 0;
    for (int64_t i = 0; i < n; ++i) nnz += lcnt[i] + 1 + ucnt[i];
    cgvk_csr* a = csr_alloc(n, nnz);
    /* row i = [lower (from rows < i, ascending) | diag | upper] */
    a->row_ptr[0] = 0;
    for (int64_t i = 0; i < n; ++i) a->row_ptr[i + 1] = a->row_ptr[i] + lcnt[i] + 1 + ucnt[i];
    int64_t* lfill = (int64_t*)calloc((size_t)n, sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i) {
        const int64_t base_up = a->row_ptr[i] + lcnt[i] + 1;
        for (int64_t c = 0; c < ucnt[i]; ++c) {
            const int64_t j = uj[i * per_row + c];
            const double v = uv[i * per_row + c];
            a->col_idx[base_up + c] = j;
            a->values[base_up + c] = v;
            const int64_t pos = a->row_ptr[j] + lfill[j]++;
            a->col_idx[pos] = i;
            a->values[pos] = v;
        }
    }
    for (int64_t i = 0; i < n; ++i) {
        const int64_t dpos = a->row_ptr[i] + lcnt[i];
        double acc = 0.0;
        for (int64_t k = a->row_ptr[i]; k < a->row_ptr[i + 1]; ++k)
            if (k != dpos) acc += fabs(a->values[k]);
        a->col_idx[dpos] = i;
        a->values[dpos] = acc + 1e-3;
    }
    for (int64_t i = 0; i < n; ++i)
        for (int64_t k = a->row_ptr[i]; k < a->row_ptr[i + 1]; ++k)
            a->values[k] = a->values[k] * (s[i] * s[a->col_idx[k]]);
    free(lfill);
    free(s);
    free(uj);
    free(uv);
    free(ucnt);
    free(lcnt);
    return a;
}

/* b = A*x with the reference's per-row left-to-right order
 * (src/sparse_matrix.cpp:109-118); input synthesis for b = A x*. */
void cgvk_gen_spmv(const cgvk_csr* a, const double* x, double* y) {
    for (int64_t i = 0; i < a->n; ++i) {
        double sum = 0.0;
        for (int64_t k = a->row_ptr[i]; k < a->row_ptr[i + 1]; ++k)
            sum += a->values[k] * x[a->col_idx[k]];
        y[i] = sum;
    }
}
