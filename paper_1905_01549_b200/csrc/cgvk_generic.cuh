// Generic device kernels: CSR upload/validation, the L1 operators behind the
// reference's spmv / block_spmv / Preconditioner / dot entry points, and the
// pieces initialize() is assembled from. Same arithmetic contract as the
// variant kernels (rounded mul/add, canonical dot tree).
#pragma once

#include "cgvk_device.cuh"

namespace cgvk {

// int64 CSR (the reference's host layout) -> int32 device CSR, checking the
// validate_csr invariants (src/sparse_matrix.cpp:64-82) on the way:
//   bit 0 row_ptr not monotone / wrong ends, bit 1 column out of range,
//   bit 2 columns not strictly increasing.
__global__ void k_convert_csr(int64_t n, int64_t ncols, int64_t nnz, const int64_t* __restrict__ rp64,
                              const int64_t* __restrict__ ci64, int* __restrict__ rp32,
                              int* __restrict__ ci32, int* flags) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int f = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += stride) {
        const int64_t a = rp64[i];
        if (i == 0 && a != 0) f |= 1;
        if (i == n && a != nnz) f |= 1;
        if (i < n) {
            const int64_t b = rp64[i + 1];
            if (b < a || a < 0 || b > nnz) f |= 1;
        }
        rp32[i] = (int)a;
    }
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += stride) {
        const int64_t c = ci64[k];
        if (c < 0 || c >= ncols) f |= 2;
        ci32[k] = (int)c;
    }
    if (f) atomicOr(flags, f);
}

// strictly increasing columns inside each row (needs a valid row_ptr)
__global__ void k_check_sorted(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                               int* flags) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        for (int k = rp[i] + 1; k < rp[i + 1]; ++k)
            if (ci[k] <= ci[k - 1]) {
                atomicOr(flags, 4);
                break;
            }
    }
}

// is_symmetric (src/sparse_matrix.cpp:84-107): every (i,j,v) has a stored
// (j,i) with identical bits (binary search in the sorted row j).
__global__ void k_check_symmetric(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                                  const double* __restrict__ va, int* flags) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        for (int k = rp[i]; k < rp[i + 1]; ++k) {
            const int j = ci[k];
            int lo = rp[j], hi = rp[j + 1] - 1, hit = -1;
            while (lo <= hi) {
                const int mid = (lo + hi) >> 1;
                if (ci[mid] == i) {
                    hit = mid;
                    break;
                }
                if (ci[mid] < i) lo = mid + 1;
                else hi = mid - 1;
            }
            if (hit < 0 || __double_as_longlong(va[hit]) != __double_as_longlong(va[k])) {
                atomicOr(flags, 8);
                return;
            }
        }
    }
}

// Preconditioner::jacobi (src/preconditioner.cpp:12-31): first stored
// diagonal entry of each row; missing or <= 0 sets flags bit 0.
__global__ void k_jacobi(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                         const double* __restrict__ va, double* __restrict__ inv_diag, int* flags) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double d = 0.0;
        bool found = false;
        for (int k = rp[i]; k < rp[i + 1]; ++k)
            if (ci[k] == i) {
                d = va[k];
                found = true;
                break;
            }
        if (!found || !(d > 0.0)) {
            atomicOr(flags, 1);
            inv_diag[i] = 0.0;
        } else {
            inv_diag[i] = DIV(1.0, d);
        }
    }
}

// y = A x, or y = b - A x when b != nullptr (the r0 / true-residual form,
// src/variants.cpp:376-377, src/diagnostics.cpp:19-21); dx: gather d∘x.
__global__ void __launch_bounds__(kBlock, kMinBlocksPerSM)
    k_spmv(Params P, const double* __restrict__ x, const double* __restrict__ b, double* y, int dx) {
    for (int tile = blockIdx.x; tile < P.ntiles; tile += gridDim.x) {
        const int i = tile * kBlock + threadIdx.x;
        if (i >= P.n) continue;
        const double sum = dx ? row_sum(P, i, [&](int j) { return MUL(__ldg(P.d + j), __ldg(x + j)); })
                              : row_sum(P, i, [&](int j) { return __ldg(x + j); });
        y[i] = b ? SUB(b[i], sum) : sum;
    }
}

__global__ void __launch_bounds__(kBlock, kMinBlocksPerSM)
    k_block_spmv(Params P, const double* __restrict__ x1, const double* __restrict__ x2, double* y1,
                 double* y2) {
    for (int tile = blockIdx.x; tile < P.ntiles; tile += gridDim.x) {
        const int i = tile * kBlock + threadIdx.x;
        if (i >= P.n) continue;
        double a, b;
        row_sum2(P, i, [&](int j) { return __ldg(x1 + j); }, [&](int j) { return __ldg(x2 + j); }, a, b);
        y1[i] = a;
        y2[i] = b;
    }
}

// out = d∘in (Preconditioner::apply, src/preconditioner.cpp:41) or a copy
__global__ void k_scale(int n, const double* __restrict__ d, const double* __restrict__ in,
                        double* __restrict__ out) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        out[i] = d ? MUL(d[i], in[i]) : in[i];
}

// out = a - b (diagnostics' gap vectors, src/diagnostics.cpp:22-31,52-57)
__global__ void k_sub(int n, const double* __restrict__ a, const double* __restrict__ b,
                      double* __restrict__ out) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        out[i] = SUB(a[i], b[i]);
}

// Three-term Lanczos recurrence residual, src/diagnostics.cpp:74-109:
// q_k = sign_k r_{k-1} / ||r_{k-1}||, then d_i = (A q_k)_i - (c_{k+1} q_{k+1,i}
// + c_k q_{k,i} + c_{k-1} q_{k-1,i}) with the same operation order.
__global__ void k_lanczos_q(int n, double sign, const double* __restrict__ r, double nrm,
                            double* __restrict__ q) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        q[i] = DIV(MUL(sign, r[i]), nrm);
}
__global__ void k_lanczos_d(int n, const double* __restrict__ lhs, const double* __restrict__ qk,
                            const double* __restrict__ rk, double sign_kp1, double n_k,
                            const double* __restrict__ rkm2, double sign_km1, double n_km2,
                            double c_kp1, double c_k, double c_km1, double* __restrict__ d) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const double q_kp1 = DIV(MUL(sign_kp1, rk[i]), n_k);
        const double q_km1 = DIV(MUL(sign_km1, rkm2[i]), n_km2);
        d[i] = SUB(lhs[i], ADD(ADD(MUL(c_kp1, q_kp1), MUL(c_k, qk[i])), MUL(c_km1, q_km1)));
    }
}

struct DotArgs {
    int n, ntiles, order;
    const double* x[4];
    const double* y[4];
    int dx[4];  // multiply x by d on the fly
    const double* d;
    double* part;
    unsigned int* counter;
    double* out;
};

// Up to four dots in the canonical order; results in out[0..ND).
template <int ND>
__global__ void __launch_bounds__(kBlock, kMinBlocksPerSM) k_dots(DotArgs A) {
    double acc[ND], tot[ND];
#pragma unroll
    for (int q = 0; q < ND; ++q) acc[q] = 0.0;
    // one CTA per virtual CTA (canonical order)
    CGVK_FOR_TILE(tile, A.order, static_cast<int>(blockIdx.x), A.ntiles, static_cast<int>(gridDim.x)) {
        const int i = tile * kBlock + threadIdx.x;
        if (i >= A.n) continue;
#pragma unroll
        for (int q = 0; q < ND; ++q) {
            const double xv = A.dx[q] ? MUL(A.d[i], A.x[q][i]) : A.x[q][i];
            acc[q] = ADD(acc[q], MUL(xv, A.y[q][i]));
        }
    }
    if (!reduce_grid<ND>(acc, A.part, A.counter, tot)) return;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int q = 0; q < ND; ++q) A.out[q] = tot[q];
    }
}

__global__ void k_set_limit(Ctrl* c, int k_limit) { c->k_limit = k_limit; }
__global__ void k_set_tol(Ctrl* c, double tol) { c->tol = tol; }

}  // namespace cgvk
