// cgvk C-ABI implementation: device matrix, solver runtime (streams, CUDA
// graphs of whole iterations, host mirror of the device control block) and
// the reference-facing entry points declared in include/cgvk.h.
#include "cgvk.h"
#include "cgvk_generic.cuh"
#include "cgvk_variants.cuh"
#include "cgvk_dist.cuh"
#include "cgvk_band.cuh"

#include <cub/device/device_scan.cuh>

#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

using namespace cgvk;

namespace {

thread_local std::string g_err;

int set_err(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CK(call)                                                                          \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess)                                                            \
            return set_err(CGVK_ECUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_),    \
                           __FILE__, __LINE__);                                           \
    } while (0)

#define TRY(expr)                  \
    do {                           \
        int rc_ = (expr);          \
        if (rc_ != CGVK_OK) return rc_; \
    } while (0)

constexpr int kMaxStageCap = 12288;  // CSR entries per stage (tiles above: direct loads)

// Experiment knobs (environment, read at matrix/solver creation).
// CGVK_DEBUG >= 2: host-side phase timings of matrix / solver creation
struct PhaseTimer {
    const char* what;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    bool on;
    explicit PhaseTimer(const char* w);
    void mark(const char* phase) {
        if (!on) return;
        const auto t = std::chrono::steady_clock::now();
        fprintf(stderr, "cgvk %s: %s %.2f ms\n", what, phase,
                std::chrono::duration<double, std::milli>(t - t0).count());
        t0 = t;
    }
};

int env_int(const char* name, int dflt) {
    const char* v = getenv(name);
    return v && *v ? atoi(v) : dflt;
}

PhaseTimer::PhaseTimer(const char* w) : what(w), on(env_int("CGVK_DEBUG", 0) >= 2) {}

int grid_elem(int64_t n) {
    int64_t g = (n + 255) / 256;
    if (g > 148 * 16) g = 148 * 16;
    return g < 1 ? 1 : (int)g;
}

// Device memory comes from the device's stream-ordered pool with an
// unlimited release threshold: after the first solve, matrix and solver
// setup reuse cached memory instead of mapping fresh pages (measured: plain
// cudaMalloc/cudaFree made one solver creation take 20-280 ms on the B200
// boxes, dominating the end-to-end time of a sweep). Allocation and free are
// ordered on a per-device pool stream; dalloc synchronises it so the memory
// is usable from any stream, and every owner synchronises its own streams
// before dfree.
cudaStream_t pool_stream() {
    static std::mutex mu;
    static cudaStream_t streams[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    if (!streams[dev]) {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        cudaStreamCreateWithFlags(&streams[dev], cudaStreamNonBlocking);
    }
    return streams[dev];
}

// Plain (cudaMalloc) allocations: the vectors of a multi-process peer-memory
// group must be IPC-shareable, which stream-ordered pool memory is not
// (cgvk_group.inc). Set per thread while such a group allocates.
bool& plain_alloc_mode() {
    static thread_local bool on = false;
    return on;
}
std::mutex& plain_mu() {
    static std::mutex mu;
    return mu;
}
std::vector<void*>& plain_set() {
    static std::vector<void*> v;
    return v;
}
int dalloc_plain(void** p, size_t bytes) {
    const cudaError_t e = cudaMalloc(p, bytes);
    if (e != cudaSuccess) {
        *p = nullptr;
        return set_err(CGVK_ENOMEM, "device allocation (%zu bytes): %s", bytes, cudaGetErrorString(e));
    }
    std::lock_guard<std::mutex> lock(plain_mu());
    plain_set().push_back(*p);
    return CGVK_OK;
}
// true if p was a plain allocation (now freed)
bool plain_release(void* p) {
    {
        std::lock_guard<std::mutex> lock(plain_mu());
        auto& v = plain_set();
        auto it = std::find(v.begin(), v.end(), p);
        if (it == v.end()) return false;
        v.erase(it);
    }
    cudaFree(p);
    return true;
}

template <class T>
int dalloc(T** p, size_t count) {
    if (count == 0) count = 1;
    if (plain_alloc_mode()) return dalloc_plain(reinterpret_cast<void**>(p), sizeof(T) * count);
    cudaStream_t st = pool_stream();
    cudaError_t e = cudaMallocAsync((void**)p, sizeof(T) * count, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
        *p = nullptr;
        return set_err(CGVK_ENOMEM, "device allocation (%zu bytes): %s", sizeof(T) * count,
                       cudaGetErrorString(e));
    }
    return CGVK_OK;
}

void dfree(void* p) {
    if (!p) return;
    if (plain_release(p)) return;
    cudaFreeAsync(p, pool_stream());
}

}  // namespace

// ===================================================================== matrix

struct cgvk_matrix_s {
    int device = 0;
    int64_t n = 0, nnz = 0;
    int ntiles = 0, gmax = 0, G = 1, sms = 0;
    int cap = 4;  // CSR entries a pipeline stage holds (max over tiles, capped)
    int64_t ncols = 0;  // == n, or n + halo for a rank-local matrix
    // row partition (rank-local matrices; a plain matrix is rank 0 of 1)
    int nranks = 1, rank = 0;
    int64_t gn = 0, glo = 0;        // global size, first global row
    int64_t nlow = 0, nup = 0;      // halo columns: [hbase, hbase+nlow) lower, [hbase+nlow, ncols) upper
    int64_t hbase = 0;              // first halo column: n rounded up to 32 (no cache line holds own rows and halo)
    int64_t nsend_lo = 0, nsend_hi = 0;
    int* send_lo = nullptr;         // local rows the lower neighbour's halo reads (sorted)
    int* send_hi = nullptr;         // local rows the upper neighbour's halo reads (sorted)
    int64_t send_lo0 = -1, send_hi0 = -1;  // first row when those rows are contiguous (z-slabs), else -1
    int order = 0;  // canonical tile order (fixed per matrix; reported to the oracle)
    int l2pol = 0;  // TMA L2 policy for the pipeline streams
    int* rp = nullptr;
    int* ci = nullptr;
    double* va = nullptr;
    // band engine copy of A (cgvk_band.cuh); band_h < 0: CSR engine
    int band_h = -1;
    int* band_off = nullptr;
    unsigned int* band_meta = nullptr;
    double* band_va = nullptr;
    unsigned short* band_ci = nullptr;
    int64_t band_entries = 0;
    double* inv_diag = nullptr;  // built on first use
    int jacobi_state = 0;        // 0 not built, 1 ok, -1 missing/non-positive diagonal
    cudaStream_t stream = nullptr;
    // L1-op scratch (guarded by mu: the matrix may be shared across threads)
    std::mutex mu;
    double* part = nullptr;
    unsigned int* counter = nullptr;
    double* out = nullptr;
    int* flags = nullptr;
    double* tmp[4] = {nullptr, nullptr, nullptr, nullptr};
    struct SpmvEngine* spmv_eng = nullptr;  // the L1 SpMV through the solver's engines (built on first use)

    Params base() const {
        Params P{};
        P.n = (int)n;
        P.ntiles = ntiles;
        P.rp = rp;
        P.ci = ci;
        P.va = va;
        P.d = inv_diag;
        P.band_off = band_off;
        P.band_meta = band_meta;
        P.band_va = band_va;
        P.band_ci = band_ci;
        P.band_h = band_h;
        P.order = order;
        P.l2pol = l2pol;
        return P;
    }
};

int matrix_create(int64_t n, int64_t ncols, const int64_t* row_ptr, const int64_t* col_idx,
                  const double* values, int device, int flags, bool check_sorted, cgvk_matrix* out);
// The L1 SpMV through the solver's engines (defined with the launch machinery below).
struct SpmvEngine;
int spmv_engine(cgvk_matrix a, int nrhs, const double* x1, const double* x2, double* y1, double* y2);
int spmv_engine_launch(cgvk_matrix a, int nrhs, const double* x1, const double* x2, double* y1, double* y2);
void free_spmv_engine(SpmvEngine* e);

namespace {

int ensure_jacobi(cgvk_matrix a) {
    if (a->jacobi_state == 1) return CGVK_OK;
    if (a->jacobi_state == -1)
        return set_err(CGVK_EINVAL, "Jacobi preconditioner needs a positive diagonal");
    if (!a->inv_diag) TRY(dalloc(&a->inv_diag, a->ncols + 32));  // (+ halo columns: PrF on a rank gathers d there)
    CK(cudaMemsetAsync(a->flags, 0, sizeof(int), a->stream));
    if (a->n > 0)
        k_jacobi<<<grid_elem(a->n), 256, 0, a->stream>>>((int)a->n, a->rp, a->ci, a->va, a->inv_diag,
                                                          a->flags);
    int flags = 0;
    CK(cudaMemcpyAsync(&flags, a->flags, sizeof(int), cudaMemcpyDeviceToHost, a->stream));
    CK(cudaStreamSynchronize(a->stream));
    a->jacobi_state = flags ? -1 : 1;
    if (flags) return set_err(CGVK_EINVAL, "Jacobi preconditioner needs a positive diagonal");
    return CGVK_OK;
}

// canonical dots of (x_q, y_q) with optional d∘x_q into dout[0..nd) on the
// device (stream-ordered, no host sync)
int launch_dots(cgvk_matrix a, cudaStream_t stream, double* part, unsigned int* counter, double* dout,
                int nd, const double* const* xs, const double* const* ys, const int* dxs) {
    DotArgs A{};
    A.n = (int)a->n;
    A.ntiles = a->ntiles;
    A.order = a->order;
    for (int q = 0; q < nd; ++q) {
        A.x[q] = xs[q];
        A.y[q] = ys[q];
        A.dx[q] = dxs ? dxs[q] : 0;
    }
    A.d = a->inv_diag;
    A.part = part;
    A.counter = counter;
    A.out = dout;
    switch (nd) {
        case 1: k_dots<1><<<a->G, kBlock, 0, stream>>>(A); break;
        case 2: k_dots<2><<<a->G, kBlock, 0, stream>>>(A); break;
        case 3: k_dots<3><<<a->G, kBlock, 0, stream>>>(A); break;
        default: k_dots<4><<<a->G, kBlock, 0, stream>>>(A); break;
    }
    CK(cudaGetLastError());
    return CGVK_OK;
}

// ... and the results to the host
int run_dots(cgvk_matrix a, cudaStream_t stream, double* part, unsigned int* counter, double* dout,
             int nd, const double* const* xs, const double* const* ys, const int* dxs,
             double* host_out) {
    if (a->n == 0) {
        for (int q = 0; q < nd; ++q) host_out[q] = 0.0;
        return CGVK_OK;
    }
    TRY(launch_dots(a, stream, part, counter, dout, nd, xs, ys, dxs));
    CK(cudaMemcpyAsync(host_out, dout, sizeof(double) * nd, cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    return CGVK_OK;
}

int ensure_tmp(cgvk_matrix a, int count) {
    for (int q = 0; q < count; ++q)
        if (!a->tmp[q]) TRY(dalloc(&a->tmp[q], a->n + 32));  // (+32: bulk copies of the last tile)
    return CGVK_OK;
}

// Band engine layout (cgvk_band.cuh): SELL-C-sigma, C = 32, sigma = 256.
// Window half-width H (tiles): every column of tile t lies in tiles
// [t - H, t + H]. Applicable to a plain (single-rank) matrix whose 16-bit
// window offsets fit and whose window rings fit in shared memory.
constexpr int kBandMaxH = 19;  // 2 operands x (2H + 2) x 2 KB <= 160 KB

// max over rows of the tile distance of the first / last column (columns are
// sorted, validated on the device before this runs)
__global__ void k_band_h(int n, const int* __restrict__ rp, const int* __restrict__ ci, int* h) {
    int m = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        if (rp[i + 1] == rp[i]) continue;
        const int t = i / kBlock, lo = ci[rp[i]] / kBlock, hi = ci[rp[i + 1] - 1] / kBlock;
        m = max(m, max(t - lo, hi - t));
    }
    if (m > 0) atomicMax(h, m);
}

int band_half_width(cgvk_matrix a) {
    CK(cudaMemsetAsync(a->flags, 0, sizeof(int), a->stream));
    k_band_h<<<grid_elem(a->n), 256, 0, a->stream>>>((int)a->n, a->rp, a->ci, a->flags);
    int h = 0;
    CK(cudaMemcpyAsync(&h, a->flags, sizeof(int), cudaMemcpyDeviceToHost, a->stream));
    CK(cudaStreamSynchronize(a->stream));
    return h > kBandMaxH ? -1 : h;
}

// One CTA per tile: rows sorted by length, descending and stable (rank =
// #longer + #equal before), meta word per slot, slot of each row, slice sizes.
__global__ void __launch_bounds__(kBlock) k_band_tiles(int n, const int* __restrict__ rp, unsigned int* meta,
                                                       int* slot_of, long long* sizes, int* flags) {
    __shared__ int len_s[kBlock];
    __shared__ int sorted_len[kBlock];
    const int t = blockIdx.x, q = threadIdx.x;
    const int r0 = t * kBlock, r = r0 + q;
    const int rows = min(kBlock, n - r0);
    const int len = q < rows ? rp[r + 1] - rp[r] : 0;
    len_s[q] = len;
    __syncthreads();
    int rank = 0;
    for (int j = 0; j < kBlock; ++j) {
        const int lj = len_s[j];
        rank += (lj > len) || (lj == len && j < q);
    }
    if (len >= (1 << 24)) atomicOr(flags, 1);
    meta[(size_t)t * kBlock + rank] = ((unsigned int)len << 8) | (unsigned int)q;
    if (q < rows) slot_of[r] = t * kBlock + rank;
    sorted_len[rank] = len;
    __syncthreads();
    if (q < kWarps) sizes[(size_t)t * kWarps + q] = 32ll * sorted_len[32 * q];  // slice 32q+.. : first is longest
}

__global__ void k_narrow_off(int count, const long long* __restrict__ off64, int* off) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x)
        off[i] = (int)off64[i];
}

// entries of row i -> its slot of the SELL-C-sigma layout
__global__ void k_fill_band(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                            const double* __restrict__ va, const int* __restrict__ slot_of,
                            const int* __restrict__ off, int H, double* bva, unsigned short* bci) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int g = slot_of[i];
        const int t = g >> 8, q = g & 255;
        const int base = off[t * kWarps + (q >> 5)] + (q & 31);
        const int wb = (t - H) * kBlock;
        for (int k = rp[i], e = 0; k < rp[i + 1]; ++k, ++e) {
            bva[base + 32 * e] = va[k];
            bci[base + 32 * e] = (unsigned short)(ci[k] - wb);
        }
    }
}

// Built on the device (a host sort of every tile cost ~200 ms on R4M).
int build_band(cgvk_matrix a, int H) {
    const int64_t n = a->n;
    const int nt = a->ntiles;
    const size_t nslice = (size_t)nt * kWarps;
    long long* sizes = nullptr;
    long long* off64 = nullptr;
    int* dslot = nullptr;
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    auto cleanup = [&]() {
        dfree(sizes);
        dfree(off64);
        dfree(dslot);
        dfree(tmp);
    };
    int rc;
    if ((rc = dalloc(&a->band_off, nslice + 16)) || (rc = dalloc(&a->band_meta, (size_t)nt * kBlock + 1)) ||
        (rc = dalloc(&sizes, nslice + 1)) || (rc = dalloc(&off64, nslice + 1)) || (rc = dalloc(&dslot, n)))
        return cleanup(), rc;
    CK(cudaMemsetAsync(a->flags, 0, sizeof(int), a->stream));
    CK(cudaMemsetAsync(sizes + nslice, 0, sizeof(long long), a->stream));
    k_band_tiles<<<nt, kBlock, 0, a->stream>>>((int)n, a->rp, a->band_meta, dslot, sizes, a->flags);
    CK(cudaGetLastError());
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, sizes, off64, (int)nslice + 1, a->stream));
    if ((rc = dalloc(reinterpret_cast<unsigned char**>(&tmp), tmp_bytes))) return cleanup(), rc;
    CK(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, sizes, off64, (int)nslice + 1, a->stream));
    long long total = 0;
    int flags = 0;
    CK(cudaMemcpyAsync(&total, off64 + nslice, sizeof(long long), cudaMemcpyDeviceToHost, a->stream));
    CK(cudaMemcpyAsync(&flags, a->flags, sizeof(int), cudaMemcpyDeviceToHost, a->stream));
    CK(cudaStreamSynchronize(a->stream));
    if (flags & 1) return cleanup(), set_err(CGVK_EINVAL, "row too long for the band engine");
    if (total >= (1ll << 31) - 64) return cleanup(), set_err(CGVK_EINVAL, "band layout exceeds 2^31 entries");
    a->band_entries = total;
    k_narrow_off<<<grid_elem(nslice + 1), 256, 0, a->stream>>>((int)nslice + 1, off64, a->band_off);
    for (int q = 1; q < 16; ++q)  // padding read by the 48-byte offset copies of the last tile
        CK(cudaMemcpyAsync(a->band_off + nslice + q, a->band_off + nslice, sizeof(int), cudaMemcpyDeviceToDevice,
                           a->stream));
    if ((rc = dalloc(&a->band_va, total + 32)) || (rc = dalloc(&a->band_ci, total + 64))) return cleanup(), rc;
    CK(cudaMemsetAsync(a->band_va, 0, sizeof(double) * (total + 32), a->stream));
    CK(cudaMemsetAsync(a->band_ci, 0, sizeof(unsigned short) * (total + 64), a->stream));
    if (n > 0)
        k_fill_band<<<grid_elem(n), 256, 0, a->stream>>>((int)n, a->rp, a->ci, a->va, dslot, a->band_off, H,
                                                          a->band_va, a->band_ci);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(a->stream);
    cleanup();
    if (e != cudaSuccess) return set_err(CGVK_ECUDA, "band layout: %s", cudaGetErrorString(e));
    a->band_h = H;
    return CGVK_OK;
}

}  // namespace

extern "C" {

const char* cgvk_last_error(void) { return g_err.c_str(); }

int cgvk_device_count(int* count) {
    CK(cudaGetDeviceCount(count));
    return CGVK_OK;
}

cgvk_variant_config cgvk_variant_config_make(int variant) {
    cgvk_variant_config c{};
    c.variant = variant;
    c.nu_expression = (variant == CGVK_M || variant == CGVK_PIPE_PR_M) ? CGVK_NU_MEURANT
                                                                       : CGVK_NU_SIMPLIFIED;
    c.recompute_nu = 1;
    c.recompute_w = 1;
    c.unsimplified_mu = 0;
    c.track_delta = 0;
    return c;
}

// src/variants.cpp:35-47
int cgvk_variant_config_validate(const cgvk_variant_config* c) {
    if (!c) return set_err(CGVK_EINVAL, "null config");
    const int v = c->variant;
    if (v < CGVK_HS || v > CGVK_PIPE_PR) return set_err(CGVK_EINVAL, "unknown variant %d", v);
    if (c->nu_expression < 0 || c->nu_expression > 2)
        return set_err(CGVK_EINVAL, "unknown nu expression %d", c->nu_expression);
    const bool pipe_pr = v == CGVK_PIPE_PR || v == CGVK_PIPE_PR_M;
    const bool predictor = v == CGVK_M || v == CGVK_PR || pipe_pr;
    if (!c->recompute_w && !pipe_pr)
        return set_err(CGVK_EINVAL, "recompute_w only applies to the pipelined PR variants");
    if (!c->recompute_nu && !predictor)
        return set_err(CGVK_EINVAL, "recompute_nu only applies to predictor variants");
    if (!predictor && c->nu_expression != CGVK_NU_SIMPLIFIED)
        return set_err(CGVK_EINVAL, "nu_expression only applies to predictor variants");
    if (c->unsimplified_mu && v != CGVK_CG_CG && v != CGVK_GV)
        return set_err(CGVK_EINVAL, "unsimplified_mu only applies to CG_CG and GV");
    if (c->track_delta && !predictor)
        return set_err(CGVK_EINVAL, "track_delta only applies to predictor variants");
    return CGVK_OK;
}

int cgvk_matrix_create_csr(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                           const double* values, int device, int flags, cgvk_matrix* out) {
    return matrix_create(n, n, row_ptr, col_idx, values, device, flags, true, out);
}

}  // extern "C"

// n rows; columns in [0, ncols) (ncols > n for a rank's local matrix, whose
// halo columns are numbered after its own rows and are therefore not sorted
// within a row — the global CSR order of the entries is what is preserved).
int matrix_create(int64_t n, int64_t ncols, const int64_t* row_ptr, const int64_t* col_idx,
                  const double* values, int device, int flags, bool check_sorted, cgvk_matrix* out) {
    if (!out) return set_err(CGVK_EINVAL, "null output handle");
    *out = nullptr;
    PhaseTimer pt("matrix_create");
    if (n < 0) return set_err(CGVK_EINVAL, "negative dimension");
    if (!row_ptr) return set_err(CGVK_EINVAL, "row_ptr length must be n+1");
    const int64_t nnz = row_ptr[n];
    if (nnz < 0) return set_err(CGVK_EINVAL, "row_ptr[n] must equal number of stored entries");
    if (n >= (int64_t(1) << 31) - 256 || nnz >= (int64_t(1) << 31))
        return set_err(CGVK_EINVAL, "device CSR uses int32 indices: n and nnz must be < 2^31");
    if (nnz > 0 && (!col_idx || !values)) return set_err(CGVK_EINVAL, "null CSR arrays");
    CK(cudaSetDevice(device));
    if (ncols < n || ncols >= (int64_t(1) << 31) - 256)
        return set_err(CGVK_EINVAL, "column count out of range");
    auto* a = new cgvk_matrix_s;
    a->device = device;
    a->n = n;
    a->ncols = ncols;
    a->hbase = n;
    a->nnz = nnz;
    a->ntiles = (int)((n + kBlock - 1) / kBlock);
    a->order = env_int("CGVK_ORDER", 0) ? 1 : 0;
    // TMA L2 policy of the matrix stream: an A that fits L2 next to the
    // solver's vectors (small problems, multi-GPU shards) is kept resident
    // (evict-last), a larger one streamed evict-first (measured P64 +3 %)
    {
        const double ws = 12.0 * (double)nnz + 4.0 * (double)n + 8.0 * 12.0 * (double)ncols;
        // one vector larger than half of L2 (V256): streamed vectors keep the
        // default policy too, only A is evict-first (measured V256 +0.8 %,
        // P128 -2.3 % — there the evict-first loads leave L2 to the vectors
        // the next kernel reads)
        const int dflt = ws < 96e6 ? 3 : 8.0 * (double)ncols > 64e6 ? 1 : 0;
        a->l2pol = env_int("CGVK_L2POL", dflt);
    }
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    a->sms = sms;
    a->gmax = sms * kVirtualPerSM;  // final value set with the engine below
    {   // stage capacity: the largest tile's CSR span (+ alignment slack for
        // the 16-bit columns' 8-entry alignment too)
        int64_t mx = 0;
        for (int64_t r0 = 0; r0 < n; r0 += kBlock) {
            const int64_t r1 = r0 + kBlock < n ? r0 + kBlock : n;
            const int64_t span = row_ptr[r1] - (row_ptr[r0] & ~int64_t(7)) + 8;
            if (span > mx) mx = span;
        }
        mx = (mx + 3) & ~int64_t(3);
        a->cap = (int)(mx < kMaxStageCap ? mx : kMaxStageCap);
    }
    a->G = a->ntiles < a->gmax ? a->ntiles : a->gmax;
    if (a->G < 1) a->G = 1;
    auto bail = [&](int rc) {
        cgvk_matrix_destroy(a);
        return rc;
    };
    int rc;
    // +padding: bulk copies round their sizes up to 16 bytes
    if ((rc = dalloc(&a->rp, n + 1 + 16)) || (rc = dalloc(&a->ci, nnz + 16)) ||
        (rc = dalloc(&a->va, nnz + 16)) ||
        (rc = dalloc(&a->part, kMaxDots * (size_t)a->gmax)) || (rc = dalloc(&a->counter, 4)) ||
        (rc = dalloc(&a->out, 8)) || (rc = dalloc(&a->flags, 1)))
        return bail(rc);
    if (cudaStreamCreateWithFlags(&a->stream, cudaStreamNonBlocking) != cudaSuccess)
        return bail(set_err(CGVK_ECUDA, "stream create failed"));
    cudaMemsetAsync(a->counter, 0, 4 * sizeof(unsigned int), a->stream);
    cudaMemsetAsync(a->flags, 0, sizeof(int), a->stream);
    // stage the int64 arrays on the device and narrow/validate there
    int64_t *rp64 = nullptr, *ci64 = nullptr;
    if ((rc = dalloc(&rp64, n + 1)) || (rc = dalloc(&ci64, nnz))) {
        dfree(rp64);
        return bail(rc);
    }
    cudaError_t e = cudaMemcpyAsync(rp64, row_ptr, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice,
                                    a->stream);
    if (e == cudaSuccess && nnz)
        e = cudaMemcpyAsync(ci64, col_idx, sizeof(int64_t) * nnz, cudaMemcpyHostToDevice, a->stream);
    if (e == cudaSuccess && nnz)
        e = cudaMemcpyAsync(a->va, values, sizeof(double) * nnz, cudaMemcpyHostToDevice, a->stream);
    if (e == cudaSuccess) {
        k_convert_csr<<<grid_elem(nnz > n ? nnz : n + 1), 256, 0, a->stream>>>(n, ncols, nnz, rp64, ci64,
                                                                              a->rp, a->ci, a->flags);
        e = cudaGetLastError();
    }
    int hflags = 0;
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(&hflags, a->flags, sizeof(int), cudaMemcpyDeviceToHost, a->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(a->stream);
    dfree(rp64);
    dfree(ci64);
    if (e != cudaSuccess) return bail(set_err(CGVK_ECUDA, "matrix upload: %s", cudaGetErrorString(e)));
    pt.mark("host scan + upload + narrow");
    if (hflags & 1) return bail(set_err(CGVK_EINVAL, "row_ptr not monotone or wrong end points"));
    if (hflags & 2) return bail(set_err(CGVK_EINVAL, "column index out of range"));
    if (n > 0) {
        if (check_sorted) k_check_sorted<<<grid_elem(n), 256, 0, a->stream>>>((int)n, a->rp, a->ci, a->flags);
        if (flags & CGVK_MATRIX_CHECK_SYMMETRIC)
            k_check_symmetric<<<grid_elem(n), 256, 0, a->stream>>>((int)n, a->rp, a->ci, a->va,
                                                                   a->flags);
        e = cudaMemcpyAsync(&hflags, a->flags, sizeof(int), cudaMemcpyDeviceToHost, a->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(a->stream);
        if (e != cudaSuccess)
            return bail(set_err(CGVK_ECUDA, "matrix validate: %s", cudaGetErrorString(e)));
        if (hflags & 4) return bail(set_err(CGVK_EINVAL, "column indices not strictly increasing"));
        if (hflags & 8) return bail(set_err(CGVK_EINVAL, "matrix is not bitwise symmetric"));
    }
    pt.mark("validate");
    // SpMV engine: band (SELL-C-sigma + shared-memory x window) for a plain
    // matrix with a narrow band and long rows, else the CSR tile pipeline.
    // Flags choose explicitly; CGVK_SPMV_ENGINE=csr|band overrides (A/B runs).
    {
        int want = (flags & CGVK_MATRIX_ENGINE_CSR) ? 0 : (flags & CGVK_MATRIX_ENGINE_BAND) ? 1 : -1;
        const char* eng = getenv("CGVK_SPMV_ENGINE");
        if (eng && strcmp(eng, "csr") == 0) want = 0;
        if (eng && strcmp(eng, "band") == 0) want = 1;
        if ((want == -1 || want == 1) && ncols == n && n > 0) {
            const bool long_rows = nnz >= (int64_t)env_int("CGVK_BAND_MIN_ROW", 16) * n;
            const int H = (want == 1 || long_rows) ? band_half_width(a) : -1;
            if (H >= 0) {
                if ((rc = build_band(a, H)) != CGVK_OK) return bail(rc);
                a->order = 1;  // the band kernels walk contiguous tile runs
            }
        }
    }
    // Canonical virtual CTAs (reduction_config): the CSR engine's kernels run
    // 3 CTAs/SM and G = 3 x SMs makes each physical CTA one virtual CTA, so
    // the grid sweeps the tiles in one monotonic pass (tile p + Gp j) and a
    // stencil's +-N^2 neighbours are still in L2 when gathered; measured
    // against 12 x SMs: V256 +7 %, P64 +14 %, P128 +0.4 %. The
    // band engine uses 6 x SMs (its SpMV kernels run 2 CTAs/SM over
    // contiguous tile runs; R4M +0.8 % vs 12 x SMs). CGVK_VPERSM overrides.
    a->gmax = sms * std::max(1, env_int("CGVK_VPERSM", a->band_h >= 0 ? kVirtualPerSMBand : kVirtualPerSMCsr));
    if (a->gmax > sms * kVirtualPerSM) return bail(set_err(CGVK_EINVAL, "CGVK_VPERSM above %d", kVirtualPerSM));
    a->G = a->ntiles < a->gmax ? a->ntiles : a->gmax;
    if (a->G < 1) a->G = 1;
    pt.mark("engine layout");
    *out = a;
    return CGVK_OK;
}

extern "C" {

int cgvk_matrix_destroy(cgvk_matrix a) {
    if (!a) return CGVK_OK;
    cudaSetDevice(a->device);
    if (a->stream) cudaStreamSynchronize(a->stream);
    dfree(a->rp);
    dfree(a->ci);
    dfree(a->va);
    dfree(a->band_off);
    dfree(a->band_meta);
    dfree(a->band_va);
    dfree(a->band_ci);
    dfree(a->inv_diag);
    dfree(a->send_lo);
    dfree(a->send_hi);
    dfree(a->part);
    dfree(a->counter);
    dfree(a->out);
    dfree(a->flags);
    for (double* t : a->tmp) dfree(t);
    free_spmv_engine(a->spmv_eng);
    if (a->stream) cudaStreamDestroy(a->stream);
    delete a;
    return CGVK_OK;
}

int cgvk_matrix_info(cgvk_matrix a, int64_t* n, int64_t* nnz, int* device) {
    if (!a) return set_err(CGVK_EINVAL, "null matrix");
    if (n) *n = a->n;
    if (nnz) *nnz = a->nnz;
    if (device) *device = a->device;
    return CGVK_OK;
}

int cgvk_matrix_engine(cgvk_matrix a, int* engine, int* band_tiles) {
    if (!a) return set_err(CGVK_EINVAL, "null matrix");
    if (engine)
        *engine = a->band_h >= 0 ? CGVK_ENGINE_BAND : CGVK_ENGINE_CSR;
    if (band_tiles) *band_tiles = a->band_h >= 0 ? a->band_h : 0;
    return CGVK_OK;
}

int cgvk_reduction_config(cgvk_matrix a, int* block, int* gmax, int* order) {
    if (!a) return set_err(CGVK_EINVAL, "null matrix");
    if (block) *block = kBlock;
    if (gmax) *gmax = a->gmax;
    if (order) *order = a->order;
    return CGVK_OK;
}

int cgvk_spmv(cgvk_matrix a, const double* x, double* y) {
    if (!a || !x || !y) return set_err(CGVK_EINVAL, "spmv dimension mismatch");
    std::lock_guard<std::mutex> lock(a->mu);
    CK(cudaSetDevice(a->device));
    if (a->n == 0) return CGVK_OK;
    if (a->ncols == a->n) return spmv_engine(a, 1, x, nullptr, y, nullptr);
    TRY(ensure_tmp(a, 2));
    CK(cudaMemcpyAsync(a->tmp[0], x, 8 * a->n, cudaMemcpyHostToDevice, a->stream));
    k_spmv<<<a->G, kBlock, 0, a->stream>>>(a->base(), a->tmp[0], nullptr, a->tmp[1], 0);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(y, a->tmp[1], 8 * a->n, cudaMemcpyDeviceToHost, a->stream));
    CK(cudaStreamSynchronize(a->stream));
    return CGVK_OK;
}

int cgvk_block_spmv(cgvk_matrix a, const double* x1, const double* x2, double* y1, double* y2) {
    if (!a || !x1 || !x2 || !y1 || !y2) return set_err(CGVK_EINVAL, "block_spmv dimension mismatch");
    std::lock_guard<std::mutex> lock(a->mu);
    CK(cudaSetDevice(a->device));
    if (a->n == 0) return CGVK_OK;
    if (a->ncols == a->n) return spmv_engine(a, 2, x1, x2, y1, y2);
    TRY(ensure_tmp(a, 4));
    CK(cudaMemcpyAsync(a->tmp[0], x1, 8 * a->n, cudaMemcpyHostToDevice, a->stream));
    CK(cudaMemcpyAsync(a->tmp[1], x2, 8 * a->n, cudaMemcpyHostToDevice, a->stream));
    k_block_spmv<<<a->G, kBlock, 0, a->stream>>>(a->base(), a->tmp[0], a->tmp[1], a->tmp[2], a->tmp[3]);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(y1, a->tmp[2], 8 * a->n, cudaMemcpyDeviceToHost, a->stream));
    CK(cudaMemcpyAsync(y2, a->tmp[3], 8 * a->n, cudaMemcpyDeviceToHost, a->stream));
    CK(cudaStreamSynchronize(a->stream));
    return CGVK_OK;
}

int cgvk_jacobi(cgvk_matrix a, double* inv_diag) {
    if (!a) return set_err(CGVK_EINVAL, "null matrix");
    std::lock_guard<std::mutex> lock(a->mu);
    CK(cudaSetDevice(a->device));
    TRY(ensure_jacobi(a));
    if (inv_diag && a->n)
        CK(cudaMemcpy(inv_diag, a->inv_diag, 8 * a->n, cudaMemcpyDeviceToHost));
    return CGVK_OK;
}

int cgvk_precond_apply(cgvk_matrix a, int kind, const double* in, double* out) {
    if (!a || !in || !out) return set_err(CGVK_EINVAL, "preconditioner dimension mismatch");
    if (kind != CGVK_PRECOND_IDENTITY && kind != CGVK_PRECOND_JACOBI)
        return set_err(CGVK_EINVAL, "unknown preconditioner kind %d", kind);
    std::lock_guard<std::mutex> lock(a->mu);
    CK(cudaSetDevice(a->device));
    if (kind == CGVK_PRECOND_JACOBI) TRY(ensure_jacobi(a));
    if (a->n == 0) return CGVK_OK;
    TRY(ensure_tmp(a, 2));
    CK(cudaMemcpyAsync(a->tmp[0], in, 8 * a->n, cudaMemcpyHostToDevice, a->stream));
    k_scale<<<grid_elem(a->n), 256, 0, a->stream>>>((int)a->n, kind ? a->inv_diag : nullptr, a->tmp[0],
                                                     a->tmp[1]);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, a->tmp[1], 8 * a->n, cudaMemcpyDeviceToHost, a->stream));
    CK(cudaStreamSynchronize(a->stream));
    return CGVK_OK;
}

int cgvk_dot(cgvk_matrix a, const double* x, const double* y, double* out) {
    if (!a || !x || !y || !out) return set_err(CGVK_EINVAL, "vector dimension mismatch");
    std::lock_guard<std::mutex> lock(a->mu);
    CK(cudaSetDevice(a->device));
    if (a->n == 0) {
        *out = 0.0;
        return CGVK_OK;
    }
    TRY(ensure_tmp(a, 2));
    CK(cudaMemcpyAsync(a->tmp[0], x, 8 * a->n, cudaMemcpyHostToDevice, a->stream));
    CK(cudaMemcpyAsync(a->tmp[1], y, 8 * a->n, cudaMemcpyHostToDevice, a->stream));
    const double* xs[1] = {a->tmp[0]};
    const double* ys[1] = {a->tmp[1]};
    return run_dots(a, a->stream, a->part, a->counter, a->out, 1, xs, ys, nullptr, out);
}

// Device-timed L1 operators for the cost-model calibration:
// CUDA events around `reps` back-to-back launches on the matrix's stream.
int cgvk_time_ops(cgvk_matrix a, int reps, double* ms) {
    if (!a || !ms || reps < 1) return set_err(CGVK_EINVAL, "null argument");
    std::lock_guard<std::mutex> lock(a->mu);
    CK(cudaSetDevice(a->device));
    for (int q = 0; q < CGVK_TIMED_OPS; ++q) ms[q] = 0.0;
    if (a->n == 0) return CGVK_OK;
    TRY(ensure_tmp(a, 4));
    const int n = (int)a->n;
    for (int q = 0; q < 4; ++q) CK(cudaMemsetAsync(a->tmp[q], 0, 8 * a->n, a->stream));
    const Params P = a->base();
    DotArgs D{};
    D.n = n;
    D.ntiles = a->ntiles;
    D.order = a->order;
    D.x[0] = a->tmp[0];
    D.y[0] = a->tmp[1];
    D.part = a->part;
    D.counter = a->counter;
    D.out = a->out;
    const bool eng = a->ncols == a->n;  // the engines' SpMV (cgvk_spmv's), else the generic kernels
    int erc = CGVK_OK;
    auto op = [&](int which) {
        switch (which) {
            case CGVK_TIME_SPMV:
                if (eng) erc = spmv_engine_launch(a, 1, a->tmp[0], nullptr, a->tmp[2], nullptr);
                else k_spmv<<<a->G, kBlock, 0, a->stream>>>(P, a->tmp[0], nullptr, a->tmp[2], 0);
                break;
            case CGVK_TIME_BLOCK_SPMV:
                if (eng) erc = spmv_engine_launch(a, 2, a->tmp[0], a->tmp[1], a->tmp[2], a->tmp[3]);
                else k_block_spmv<<<a->G, kBlock, 0, a->stream>>>(P, a->tmp[0], a->tmp[1], a->tmp[2], a->tmp[3]);
                break;
            case CGVK_TIME_DOT: k_dots<1><<<a->G, kBlock, 0, a->stream>>>(D); break;
            default: k_scale<<<grid_elem(n), 256, 0, a->stream>>>(n, nullptr, a->tmp[0], a->tmp[2]); break;
        }
    };
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    for (int which = 0; which < CGVK_TIMED_OPS; ++which) {
        op(which);  // warm-up
        CK(cudaEventRecord(e0, a->stream));
        for (int r = 0; r < reps; ++r) op(which);
        CK(cudaEventRecord(e1, a->stream));
        CK(cudaEventSynchronize(e1));
        TRY(erc);
        float f = 0.f;
        CK(cudaEventElapsedTime(&f, e0, e1));
        ms[which] = f / reps;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    CK(cudaGetLastError());
    return CGVK_OK;
}

// CGVK_TIMELINE builds only (A/B experiments): the per-CTA phase stamps of
// the last update (0) and SpMV (1) kernel launches, [2][1024][8] ns.
int cgvk_debug_timeline(unsigned long long* out) {
#if CGVK_TIMELINE
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpyFromSymbol(out, g_timeline, sizeof(g_timeline)));
    static unsigned long long zeros[2 * 1024 * 8] = {};  // read-and-clear
    CK(cudaMemcpyToSymbol(g_timeline, zeros, sizeof(g_timeline)));
    return CGVK_OK;
#else
    (void)out;
    return set_err(CGVK_EINVAL, "built without CGVK_TIMELINE");
#endif
}

int cgvk_host_register(void* ptr, uint64_t bytes) {
    CK(cudaHostRegister(ptr, bytes, cudaHostRegisterDefault));
    return CGVK_OK;
}

int cgvk_host_unregister(void* ptr) {
    CK(cudaHostUnregister(ptr));
    return CGVK_OK;
}

}  // extern "C"

// ===================================================================== solver

using StreamFn = void (*)(Params, StageCfg);
using FinalizeFn = void (*)(Params, const double*, int);

// One pipelined kernel: function, stage configuration, grid, dynamic smem.
struct KLaunch {
    StreamFn fn = nullptr;
    StreamFn fn_peer = nullptr;  // the peer-memory rank form of fn (null: none)
    StageCfg S{};
    int grid = 1;
    int threads = kThreads;
    size_t smem = 0;
};

struct cgvk_solver_s {
    cgvk_matrix a = nullptr;
    cgvk_variant_config cfg{};
    int prec = 0;
    int64_t n = 0;
    cudaStream_t stream = nullptr;
    double *x = nullptr, *r = nullptr, *p0 = nullptr, *p1 = nullptr, *s = nullptr, *w = nullptr,
           *u = nullptr, *t = nullptr, *rt = nullptr, *st = nullptr, *wt = nullptr, *b = nullptr,
           *tmp = nullptr;
    double* wpred = nullptr;  // run() with probes on a pipelined PR variant
    double* slab = nullptr;   // backs every vector above and part / hist / dout / counter / ctrl
    double *part = nullptr, *hist = nullptr, *dout = nullptr;
    unsigned int* counter = nullptr;
    int hist_cap = 0;
    Ctrl* ctrl = nullptr;
    Ctrl mirror{};
    bool mirror_fresh = true;
    int k_target = 0;
    KLaunch k1, k2;
    KLaunch k1c0, k1c, k2c, kt;  // chained schedule (graphs): see chain_prologue
    // One kernel per iteration (PrF, cgvk_variants.cuh: PR / M on a problem
    // that fits L2): k1 = k2 = that kernel, even and odd launches alternate
    // the control-block / partial copies, kt_odd closes a graph with an odd
    // number of them; s2 / g2 are the second buffers of s and r~ (or r).
    int fused = 0;  // 0: two kernels per iteration; 1: PrF; 2: CgF; 3: GvF; 4: PprF
    KLaunch kt_odd;
    double *s2 = nullptr, *g2 = nullptr;          // PrF
    double *r2 = nullptr, *w2 = nullptr;          // CgF (s2 too)
    double *u2 = nullptr, *t2 = nullptr;          // GvF (w2 too; owned: b0 / b1 / b2)
    double *a2 = nullptr;                         // PprF: s~ | s (g2 = r~ | r, w2, u2 too)
    double *b0 = nullptr, *b1 = nullptr, *b2 = nullptr;
    cudaGraphExec_t g8 = nullptr;  // the gn-iteration graph (a remainder goes out as plain launches)
    int gn = 8;
    Params P{};
    int allocated = 0;
    // row-partitioned solve (cgvk_group_create): this rank's share
    struct Group* group = nullptr;
    std::shared_ptr<struct Group> group_ref;  // keeps the group alive while a member lives
    bool owns_stream = true;
    double *rank_tot = nullptr, *all_tot = nullptr;
    double *sbuf_lo = nullptr, *sbuf_hi = nullptr, *rbuf_lo = nullptr, *rbuf_hi = nullptr;
    FinalizeFn fin1 = nullptr, fin2 = nullptr;
    unsigned int* p2p_err = nullptr;  // peer-memory rank: the window's give-up flag (cgvk_group.inc)
};

namespace {

constexpr int kSmemPerSM = 227 * 1024;

// Physical CTAs for Gv virtual CTAs with `cap` resident: every physical CTA
// runs the same number of virtual CTAs (when Gv allows it).
int balanced_grid(int Gv, int cap) {
    if (cap >= Gv) return Gv;
    const int per = (Gv + cap - 1) / cap;
    return (Gv + per - 1) / per;
}

// The dynamic shared-memory attribute is per function: only ever raise it
// (solvers of other matrices may already have launches captured with more).
int raise_smem(const void* fn, size_t bytes) {
    static std::mutex mu;
    static std::vector<std::pair<const void*, size_t>> set;
    std::lock_guard<std::mutex> lock(mu);
    size_t* cur = nullptr;
    for (auto& e : set)
        if (e.first == fn) cur = &e.second;
    if (!cur) {
        set.emplace_back(fn, 0);
        cur = &set.back().second;
    }
    if (bytes > *cur) {
        CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
        *cur = bytes;
    }
    return CGVK_OK;
}

// Band engine launch (cgvk_band.cuh): NS-stage ring for meta + per-row
// vectors, a window ring of 2H + NS tiles per gathered operand, the per-row
// contribution buffers; grid = resident CTAs (<= Gv). Knobs (experiments):
// CGVK_BAND_NSTAGE, CGVK_BAND_PF (L2 prefetch distance in tiles).
template <class Op, class Prev>
int make_band(cgvk_matrix a, KLaunch* L) {
    using Shape = BandShape<Op>;
    L->fn = k_band<Op, Prev>;
    L->threads = Shape::THREADS;
    StageCfg S{};
    S.nvec = Op::NV + Shape::NRAW;
    S.stage_bytes = band_stage_bytes(S.nvec);
    S.gvirt = a->G;
    const int ns_default = 2 * Shape::GROUPS;  // measured R4M: GV K2 350 us at 2 vs 375 at 4; pipe-PR 344 at 4 vs 372 at 8
    S.nstage = std::min(std::max(env_int("CGVK_BAND_NSTAGE", ns_default), 2), kMaxStages);
    // raw windows are filled NS - 1 tiles ahead by the producer; a combined
    // window one tile ahead by the consumers
    // (XF: a combined tile is overwritten only after the slowest warp is done
    // with it — it may trail the others by CGVK_BAND_SLACK tiles)
    S.ring = 2 * a->band_h + (Shape::XF ? 1 + kBandXfAhead + CGVK_BAND_SLACK : S.nstage);
    S.pf = std::max(env_int("CGVK_BAND_PF", 0), 0);  // measured: L2 bulk prefetch of the slices slows R4M
    const int header = ((int)sizeof(PipeHeader) + 127) & ~127;
    L->smem = (size_t)header + (size_t)S.nstage * S.stage_bytes + (size_t)Shape::NWIN * S.ring * kBlock * 8 +
              (size_t)2 * Op::ND * kBlock * 8;
    if (L->smem > (size_t)kSmemPerSM - 1024) return set_err(CGVK_EINVAL, "band window exceeds shared memory");
    TRY(raise_smem((const void*)L->fn, L->smem));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, L->fn, L->threads, L->smem));
    if (occ < 1) return set_err(CGVK_ECUDA, "band kernel does not fit on an SM");
#if CGVK_BAND_MAXNREG
    // the register-capped form where it keeps the occupancy (the register
    // file is split over 4 SM sub-partitions: two 9-warp CTAs need <= 96
    // registers; measured R4M with the slack hand-over: CG K2 262 -> 252 us
    // capped at 2 CTAs/SM, HS / PR K2 284 / 270 -> 450 / 424 us capped at 1)
    if constexpr (Shape::MINB == 2 && Shape::THREADS == kThreads && Op::ND > 0) {
        const StreamFn nr = k_band_nr<Op, Prev>;
        TRY(raise_smem((const void*)nr, L->smem));
        int occ_nr = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_nr, nr, L->threads, L->smem));
        if (occ_nr >= occ && !env_int("CGVK_BAND_NO_NR", 0)) L->fn = nr;
    }
#endif
    L->grid = balanced_grid(a->G, occ * a->sms);
    L->S = S;
    if (env_int("CGVK_DEBUG", 0))
        fprintf(stderr, "cgvk launch %s: occ %d/SM grid %d smem %zu ring %d tiles\n", __func__, occ, L->grid,
                L->smem, S.ring);
    return CGVK_OK;
}

// Configure k_stream<Op> for matrix `a`: ring depth chosen so two CTAs fit
// per SM when the stages allow it, physical grid = resident CTAs (<= Gv).
// The SpMV kernels of a band-engine matrix run k_band instead. Tuning knobs
// (experiments): CGVK_NSTAGE[_SPMV] = ring depth, CGVK_SMEM_CTAS[_SPMV] = CTAs
// per SM the stage budget targets.
template <class Op, class Prev>
int make_launch(cgvk_matrix a, KLaunch* L) {
    if constexpr (Op::CSR && !NoBand<Op>::value) {
        if (a->band_h >= 0) return make_band<Op, Prev>(a, L);
    }
    constexpr int kMinb = MinbOf<Op>::value;
    L->fn = k_stream<Op, Prev>;
    // (the peer form of a one-kernel iteration spills under the 3-CTA register
    // cap, and rank shards are small: budget for 2 CTAs)
    constexpr int kMinbPeer = HasEarlyPcur<Op>::value ? 2 : kMinb;
    if constexpr (!NoPeer<Op>::value) L->fn_peer = k_stream<Op, Prev, kMinbPeer, true>;
    // register-capped build of an Op that has one (GV / pipe-PR K1: 72
    // registers, 3 CTAs/SM): only when the working set fits L2 and the
    // virtual CTAs outnumber two CTAs per SM (measured P64 GV 18.4 -> 17.5 us,
    // pipe-PR 19.4 -> 18.8; P2D, whose 256 tiles fit either grid, and P128 /
    // V256 are slower with it)
    if constexpr (MaxnregOf<Op>::value > 0)
        if ((a->l2pol == 3 && a->G > 2 * a->sms) || env_int("CGVK_K1_NR", 0)) {
            L->fn = k_stream_nr<Op, Prev>;  // (the peer form keeps its registers: it spills under the cap)
        }
    L->threads = kThreads;
    StageCfg S{};
    S.nvec = Op::NV;
    S.cap = Op::CSR ? a->cap : 0;
    const int header = ((int)sizeof(PipeHeader) + 127) & ~127;
    if (Op::CSR) {  // two stages must fit one CTA: tiles beyond the capacity go direct
        while (S.cap > 64 &&
               header + 2 * ((stage_bytes_for(S.cap, S.nvec, true) + 127) & ~127) > kSmemPerSM - 1024)
            S.cap = (S.cap - S.cap / 8) & ~7;
    }
    S.stage_bytes = (stage_bytes_for(S.cap, S.nvec, Op::CSR) + 127) & ~127;
    S.gvirt = a->G;
    // stage budget: the SpMV kernels target CGVK_SPMV_MIN_CTAS resident CTAs,
    // the update kernels two
    // (update kernels: 3, so that every CSR-engine kernel that the register
    // budget allows runs one CTA per canonical virtual CTA, G = 3 x SMs)
    int ctas = env_int(Op::CSR ? "CGVK_SMEM_CTAS_SPMV" : "CGVK_SMEM_CTAS",
                       SmemCtasOf<Op>::value > 0 ? SmemCtasOf<Op>::value : Op::CSR ? CGVK_SPMV_MIN_CTAS : 3);
    if (Op::CSR && header + 2 * S.stage_bytes > kSmemPerSM / 2 - 2048) {
        // long rows: a 2-stage ring fills the SM -> one CTA with the full
        // register file (see k_stream's MINB)
        L->fn = k_stream<Op, Prev, 1>;
        if constexpr (!NoPeer<Op>::value) L->fn_peer = k_stream<Op, Prev, 1, true>;
        ctas = 1;
    }
    const int budget = kSmemPerSM / ctas - 2048;
    int ns = (budget - header) / S.stage_bytes;
    if (ns < 2) ns = 2;
    if (ns > 6) ns = 6;
    if (StagesOf<Op>::value >= 2 && StagesOf<Op>::value < ns) ns = StagesOf<Op>::value;
    const int forced = env_int(Op::CSR ? "CGVK_NSTAGE_SPMV" : "CGVK_NSTAGE", 0);
    if (forced >= 2 && forced <= kMaxStages) ns = forced;
    S.nstage = ns;
    L->smem = (size_t)header + (size_t)ns * S.stage_bytes;
    if (L->smem > (size_t)kSmemPerSM - 1024)
        return set_err(CGVK_EINVAL, "pipeline stage (%d bytes) exceeds shared memory", S.stage_bytes);
    TRY(raise_smem((const void*)L->fn, L->smem));
    if (L->fn_peer) TRY(raise_smem((const void*)L->fn_peer, L->smem));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, L->fn, kThreads, L->smem));
    if (occ < 1) return set_err(CGVK_ECUDA, "pipeline kernel does not fit on an SM");
    L->grid = balanced_grid(a->G, occ * a->sms);
    L->S = S;
    if (env_int("CGVK_DEBUG", 0))
        fprintf(stderr, "cgvk launch %s: occ %d/SM grid %d smem %zu nstage %d stage %d B\n", __func__, occ,
                L->grid, L->smem, S.nstage, S.stage_bytes);
    return CGVK_OK;
}

template <class Op1, class Op2>
int pick_pair(cgvk_matrix a, cgvk_solver s) {
    TRY((make_launch<Op1, Op2>(a, &s->k1)));
    TRY((make_launch<Op2, Op1>(a, &s->k2)));
    // chained schedule (chain_prologue): K1 first in a graph, K1 folding the
    // previous K2, K2 folding K1, and the graph's closing tail
    s->k1c0 = s->k1;
    s->k1c0.S.chain = CH_ON;
    s->k1c = s->k1;
    s->k1c.S.chain = CH_ON | CH_FOLD;
    s->k1c.S.gprev = s->k2.S.gvirt;
    s->k2c = s->k2;
    s->k2c.S.chain = CH_ON | CH_FOLD | CH_ODD;
    s->k2c.S.gprev = s->k1.S.gvirt;
    s->kt = KLaunch{};
    s->kt.fn = k_chain_tail<Op1, Op2>;
    s->kt.fn_peer = k_chain_tail<Op1, Op2, true>;
    s->kt.grid = 1;
    s->kt.threads = kConsumers;
    s->kt.smem = 0;
    s->kt.S = s->k2.S;
    s->kt.S.gprev = s->k2.S.gvirt;
    s->fin1 = k_finalize<Op1>;
    s->fin2 = k_finalize<Op2>;
    return CGVK_OK;
}

// One kernel per iteration, chained with itself: even launches read `ctrl` /
// `part` and write the _b copies, odd launches (CH_ODD) the reverse.
template <class Op>
int pick_fused(cgvk_matrix a, cgvk_solver s) {
    TRY((make_launch<Op, Op>(a, &s->k1)));
    s->k2 = s->k1;
    s->k1c0 = s->k1;
    s->k1c0.S.chain = CH_ON;
    s->k1c = s->k1;
    s->k1c.S.chain = CH_ON | CH_FOLD;
    s->k1c.S.gprev = s->k1.S.gvirt;
    s->k2c = s->k1c;
    s->k2c.S.chain = CH_ON | CH_FOLD | CH_ODD;
    s->kt = KLaunch{};
    s->kt.fn = k_chain_tail<Op, Op>;
    if constexpr (!NoPeer<Op>::value) s->kt.fn_peer = k_chain_tail<Op, Op, true>;
    s->kt.grid = 1;
    s->kt.threads = kConsumers;
    s->kt.smem = 0;
    s->kt.S = s->k1.S;
    s->kt.S.gprev = s->k1.S.gvirt;
    s->kt_odd = s->kt;
    s->kt_odd.S.chain = CH_ODD;
    s->fin1 = s->fin2 = k_finalize<Op>;
    return CGVK_OK;
}

template <bool PREC>
int pick_kernels(cgvk_matrix a, int v, cgvk_solver s) {
    if (s->fused == 1) return pick_fused<PrF<PREC>>(a, s);
    if (s->fused == 2) return pick_fused<CgF<PREC>>(a, s);
    if (s->fused == 3) return pick_fused<GvF<PREC>>(a, s);
    if (s->fused == 4) return pick_fused<PprF<PREC>>(a, s);
    switch (v) {
        case CGVK_HS: return pick_pair<HsK1<PREC>, HsK2<PREC>>(a, s);
        case CGVK_CG_CG: return pick_pair<CgK1<PREC>, CgK2<PREC>>(a, s);
        case CGVK_M:
        case CGVK_PR: return pick_pair<PrK1<PREC>, PrK2<PREC>>(a, s);
        case CGVK_GV: return pick_pair<GvK1<PREC>, GvK2<PREC>>(a, s);
        default: return pick_pair<PprK1<PREC>, PprK2<PREC>>(a, s);
    }
}

cudaError_t launch(cgvk_solver s, const KLaunch& L);

// the reference's allocated_vectors() (src/variants.cpp:97-103) for the
// vectors initialize() resizes (src/variants.cpp:354-444)
int ref_allocated(int v, bool prec) {
    int c = 4;  // x r p s
    if (prec) c += 1;  // r~
    const bool needs_st = prec && v != CGVK_HS && v != CGVK_CG_CG;
    if (needs_st) c += 1;
    switch (v) {
        case CGVK_CG_CG: c += 1; break;                          // w
        case CGVK_GV: c += 3 + (prec ? 1 : 0); break;            // w u t (+w~)
        case CGVK_PIPE_PR:
        case CGVK_PIPE_PR_M: c += 2 + (prec ? 2 : 0); break;     // w u (+w~ u~)
        default: break;
    }
    return c;
}

// Pipeline kernels go out with programmatic stream serialization (PDL): each
// may start its prologue (barrier init, matrix prefetch) while the previous
// kernel drains, and synchronises with griddepcontrol.wait before reading its
// results. CGVK_PDL=0 turns it off (for A/B measurements).
cudaError_t launch_with(cudaStream_t st, const KLaunch& L, const Params& P);

cudaError_t launch(cgvk_solver s, const KLaunch& L) { return launch_with(s->stream, L, s->P); }

cudaError_t launch_with(cudaStream_t st, const KLaunch& L, const Params& P) {
    // measured (profiles/r01): PDL gains 3-5 % on every variant; HS's kernels
    // signal their dependents late (PdlLate), else HS loses ~10 % to it
    static const int pdl_env = env_int("CGVK_PDL", -1);
    const bool pdl = pdl_env >= 0 ? pdl_env != 0 : true;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(L.grid);
    cfg.blockDim = dim3(L.threads);
    cfg.dynamicSmemBytes = L.smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, L.fn, P, L.S);
}

}  // namespace

// The L1 SpMV of the C ABI through the solver's engines (the CSR tile
// pipeline or the band engine, whichever the matrix uses): SpmvOp<1> / <2>.
struct SpmvEngine {
    KLaunch L[3];  // 1 and 2 right-hand sides; the residual form b - A x
};

void free_spmv_engine(SpmvEngine* e) { delete e; }

// a->mu held
int spmv_engine_launch(cgvk_matrix a, int nrhs, const double* x1, const double* x2, double* y1, double* y2) {
    if (!a->spmv_eng) {
        auto* e = new SpmvEngine;
        int rc = make_launch<SpmvOp<1>, SpmvOp<1>>(a, &e->L[0]);
        if (rc == CGVK_OK) rc = make_launch<SpmvOp<2>, SpmvOp<2>>(a, &e->L[1]);
        if (rc == CGVK_OK) rc = make_launch<SpmvOp<1, true>, SpmvOp<1, true>>(a, &e->L[2]);
        if (rc != CGVK_OK) {
            delete e;
            return rc;
        }
        a->spmv_eng = e;
    }
    if (nrhs == 0) return CGVK_OK;  // (build only)
    Params P = a->base();
    P.w = const_cast<double*>(x1);
    P.u = const_cast<double*>(x2);
    P.t = y1;
    P.s = y2;
    CK(launch_with(a->stream, a->spmv_eng->L[nrhs - 1], P));
    return CGVK_OK;
}

// host vectors in and out (cgvk_spmv / cgvk_block_spmv); a->mu held
int spmv_engine(cgvk_matrix a, int nrhs, const double* x1, const double* x2, double* y1, double* y2) {
    TRY(ensure_tmp(a, 4));
    CK(cudaMemcpyAsync(a->tmp[0], x1, 8 * a->n, cudaMemcpyHostToDevice, a->stream));
    if (nrhs == 2) CK(cudaMemcpyAsync(a->tmp[1], x2, 8 * a->n, cudaMemcpyHostToDevice, a->stream));
    TRY(spmv_engine_launch(a, nrhs, a->tmp[0], a->tmp[1], a->tmp[2], a->tmp[3]));
    CK(cudaMemcpyAsync(y1, a->tmp[2], 8 * a->n, cudaMemcpyDeviceToHost, a->stream));
    if (nrhs == 2) CK(cudaMemcpyAsync(y2, a->tmp[3], 8 * a->n, cudaMemcpyDeviceToHost, a->stream));
    CK(cudaStreamSynchronize(a->stream));
    return CGVK_OK;
}

namespace {

// The chained schedule is the default for graphs; CGVK_CHAIN=0 captures the
// last-CTA schedule instead (A/B). Row-partitioned ranks never chain (their
// reductions finish in k_finalize after the exchange).
bool use_chain() {
    static const int v = env_int("CGVK_CHAIN", 1);
    return v != 0;
}

// Iterations per long graph (step(n) replays n / gn of them, then 1-iteration
// graphs); CGVK_GRAPH_ITERS overrides.
int graph_iters() {
    static const int v = env_int("CGVK_GRAPH_ITERS", 8);
    return v < 2 ? 2 : v > 256 ? 256 : v;
}

int capture(cgvk_solver s, int iters, cudaGraphExec_t* exec) {
    CK(cudaStreamBeginCapture(s->stream, cudaStreamCaptureModeThreadLocal));
    cudaError_t e = cudaSuccess;
    if (use_chain()) {
        if (s->fused) {
            for (int i = 0; i < iters && e == cudaSuccess; ++i)
                e = launch(s, i == 0 ? s->k1c0 : (i & 1) ? s->k2c : s->k1c);
            if (e == cudaSuccess) e = launch(s, (iters & 1) ? s->kt_odd : s->kt);
        } else {
            for (int i = 0; i < iters && e == cudaSuccess; ++i) {
                e = launch(s, i ? s->k1c : s->k1c0);
                if (e == cudaSuccess) e = launch(s, s->k2c);
            }
            if (e == cudaSuccess) e = launch(s, s->kt);
        }
    } else {
        for (int i = 0; i < iters && e == cudaSuccess; ++i) {
            e = launch(s, s->k1);
            if (e == cudaSuccess && !s->fused) e = launch(s, s->k2);
        }
    }
    cudaGraph_t g = nullptr;
    const cudaError_t e_end = cudaStreamEndCapture(s->stream, &g);  // always leave capture mode
    struct GraphGuard {
        cudaGraph_t g;
        ~GraphGuard() { if (g) cudaGraphDestroy(g); }
    } guard{g};
    CK(e);
    CK(e_end);
    CK(cudaGraphInstantiate(exec, g, 0));
    // upload now (stream-ordered, off the first step()'s critical path)
    if (env_int("CGVK_GRAPH_UPLOAD", 1)) CK(cudaGraphUpload(*exec, s->stream));
    return CGVK_OK;
}

// `iters` iterations outside a graph: the kernels a graph of that length
// would hold — one chained run with one closing tail — launched on the
// solver's stream (step(n)'s remainder n % gn: a second graph per solver cost
// 0.06 ms of every solver creation to capture and instantiate, more than the
// launches it saves a short solve).
int launch_chain(cgvk_solver s, int iters) {
    if (iters <= 0) return CGVK_OK;
    if (!use_chain()) {
        for (int i = 0; i < iters; ++i) {
            CK(launch(s, s->k1));
            if (!s->fused) CK(launch(s, s->k2));
        }
        return CGVK_OK;
    }
    if (s->fused) {
        for (int i = 0; i < iters; ++i) CK(launch(s, i == 0 ? s->k1c0 : (i & 1) ? s->k2c : s->k1c));
        CK(launch(s, (iters & 1) ? s->kt_odd : s->kt));
    } else {
        for (int i = 0; i < iters; ++i) {
            CK(launch(s, i ? s->k1c : s->k1c0));
            CK(launch(s, s->k2c));
        }
        CK(launch(s, s->kt));
    }
    return CGVK_OK;
}

int refresh_mirror(cgvk_solver s) {
    CK(cudaMemcpyAsync(&s->mirror, s->ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, s->stream));
    unsigned int err = 0;
    if (s->p2p_err) CK(cudaMemcpyAsync(&err, s->p2p_err, sizeof err, cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    if (err) return set_err(CGVK_ECUDA, "peer-memory exchange: a wait for a neighbour gave up");
    s->mirror_fresh = true;
    return CGVK_OK;
}

// host forms of settle_nonpositive / settle_mu for the row-partitioned
// initialize (cgvk_group.inc), whose reductions are folded on the host
bool host_settle_nonpositive(Ctrl& c, double value, int reason, double rr) {
    if (!std::isfinite(value)) {
        c.state = ST_BREAKDOWN;
        c.reason = BR_NONFINITE;
        return true;
    }
    if (value > 0.0) return false;
    if (value == 0.0 && rr == 0.0) {
        c.state = ST_CONVERGED;
        c.criterion = CB_ZERO;
    } else {
        c.state = ST_BREAKDOWN;
        c.reason = reason;
    }
    return true;
}

bool host_settle_mu(Ctrl& c) {
    if (!std::isfinite(c.sc[SMU])) {
        c.state = ST_BREAKDOWN;
        c.reason = BR_NONFINITE;
        return true;
    }
    if (c.sc[SMU] <= 0.0) {
        c.state = ST_BREAKDOWN;
        c.reason = BR_MU;
        return true;
    }
    return false;
}

// ---------------------------------------------------------- initialize()
// src/variants.cpp:354-444 as a stream-ordered sequence: generic kernels for
// the vectors, canonical dot kernels into `dout`, and one-thread kernels that
// run the reference's scalar logic and checks on those results in the control
// block. Nothing waits for the host, so a solver is created while the
// previous solver (or the matrix upload) is still running. The reference
// returns early when a check settles the status (nu0 <= 0 after the first
// reduction, mu0 <= 0 after the second): here every kernel is enqueued
// anyway, the control block records the stage the status settled at
// (Ctrl::init_stage), and k_init_fixup restores the vectors the reference
// never computed to zero, so the state is exactly the reference's.

__global__ void k_init_ctrl(Ctrl* c, Ctrl c0) { *c = c0; }

// after <r~,r>, <r,r>, <b,b> (src/variants.cpp:382-383)
__global__ void k_init_nu(Ctrl* c, const double* __restrict__ dout, double* hist, int prec) {
    const double nu0 = dout[0], rr0 = dout[1];
    c->rr = rr0;
    c->bnorm = sqrt(dout[2]);
    if (hist) hist[0] = rr0;
    c->sc[SNU] = nu0;
    c->stats[STAT_SPMV] = 1;
    c->stats[STAT_PREC] = prec;
    c->stats[STAT_RED] = 1;
    if (settle_nonpositive(c, nu0, BR_NU, rr0)) c->init_stage = 1;
}

// after mu0 = <p0, s0> (src/variants.cpp:385-389)
__global__ void k_init_mu(Ctrl* c, const double* __restrict__ dout, int st_apply) {
    if (c->state != ST_RUNNING) return;
    c->stats[STAT_SPMV] += 1;
    c->stats[STAT_RED] += 1;
    c->sc[SMU] = dout[0];
    if (settle_mu(c)) {
        c->init_stage = 2;
        return;
    }
    c->sc[SA] = DIV(c->sc[SNU], c->sc[SMU]);
    c->stats[STAT_PREC] += st_apply;  // s~ = M s (needs_s_tilde)
}

struct InitExtras {
    int nd;            // dots in dout
    int slot[3];       // their scalar slots
    int spmv, prec;    // counter increments of the per-variant extras
};

// the per-variant extras (src/variants.cpp:396-440)
__global__ void k_init_extras(Ctrl* c, const double* __restrict__ dout, InitExtras e) {
    if (c->state != ST_RUNNING) return;
    for (int q = 0; q < e.nd; ++q) c->sc[e.slot[q]] = dout[q];
    c->stats[STAT_SPMV] += e.spmv;
    c->stats[STAT_PREC] += e.prec;
    c->stats[STAT_RED] += e.nd;
}

struct InitVecs {
    double* after_nu[2];  // computed after the nu0 check: p0, s
    double* after_mu[4];  // after the mu0 check: s~, w, u, w~ (as the variant has them)
};

__global__ void k_init_fixup(int n, const Ctrl* __restrict__ c, InitVecs v) {
    const int stage = c->init_stage;
    if (stage == 0) return;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        if (stage == 1) {
#pragma unroll
            for (int q = 0; q < 2; ++q)
                if (v.after_nu[q]) v.after_nu[q][i] = 0.0;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (v.after_mu[q]) v.after_mu[q][i] = 0.0;
    }
}

// Host-to-device uploads of solver creations are issued in creation order
// per device: a solver's b / x0 copies wait for the previous solver's, so the
// first solver starts computing after its own inputs instead of sharing the
// copy engine with every later one.
int order_uploads(cgvk_solver s, bool done) {
    static std::mutex mu;
    static cudaEvent_t last[64] = {};
    const int dev = s->a->device;
    std::lock_guard<std::mutex> lock(mu);
    if (!done) {
        if (last[dev]) CK(cudaStreamWaitEvent(s->stream, last[dev], 0));
        return CGVK_OK;
    }
    if (!last[dev]) CK(cudaEventCreateWithFlags(&last[dev], cudaEventDisableTiming));
    CK(cudaEventRecord(last[dev], s->stream));
    return CGVK_OK;
}

int solver_init(cgvk_solver s, const double* b, const double* x0) {
    cgvk_matrix a = s->a;
    const int64_t n = s->n;
    const int v = s->cfg.variant;
    const bool prec = s->prec;
    const bool stores_rt = prec;  // every variant keeps r~ in a buffer when preconditioned
    const bool needs_st = prec && v != CGVK_HS && v != CGVK_CG_CG;
    const bool pipe = v == CGVK_PIPE_PR || v == CGVK_PIPE_PR_M;
    cudaStream_t st = s->stream;
    Params P = a->base();
    const int G = a->G;
    const int eg = grid_elem(n);
    const double* d = a->inv_diag;
    Ctrl c0{};
    c0.state = ST_RUNNING;
    c0.hist_cap = s->hist_cap;
    k_init_ctrl<<<1, 1, 0, st>>>(s->ctrl, c0);

    TRY(order_uploads(s, false));
    CK(cudaMemcpyAsync(s->b, b, 8 * n, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(s->x, x0, 8 * n, cudaMemcpyHostToDevice, st));
    TRY(order_uploads(s, true));
    // y = A x through the engines' SpMV for a plain matrix (the generic kernel
    // for a rank-local one)
    const bool eng = a->ncols == a->n;
    if (eng) {
        std::lock_guard<std::mutex> lock(a->mu);
        TRY(spmv_engine_launch(a, 0, nullptr, nullptr, nullptr, nullptr));  // (builds it; launches nothing)
    }
    auto spmv = [&](const double* src, const double* bvec, double* dst) -> int {
        if (eng) {
            Params Q = P;
            Q.w = const_cast<double*>(src);
            Q.u = const_cast<double*>(bvec);
            Q.t = dst;
            CK(launch_with(st, a->spmv_eng->L[bvec ? 2 : 0], Q));
        } else {
            k_spmv<<<G, kBlock, 0, st>>>(P, src, bvec, dst, 0);
        }
        return CGVK_OK;
    };
    // r0 = b - A x0
    TRY(spmv(s->x, s->b, s->r));
    if (stores_rt) k_scale<<<eg, 256, 0, st>>>((int)n, d, s->r, s->rt);
    const double* rtv = stores_rt ? s->rt : s->r;
    {
        const double* xs[3] = {rtv, s->r, s->b};
        const double* ys[3] = {s->r, s->r, s->b};
        const int dx[3] = {0, 0, 0};
        TRY(launch_dots(a, st, s->part, s->counter, s->dout, 3, xs, ys, dx));
    }
    k_init_nu<<<1, 1, 0, st>>>(s->ctrl, s->dout, s->hist, prec ? 1 : 0);
    // p0 = r~0; s0 = A p0; mu0; alpha0
    k_scale<<<eg, 256, 0, st>>>((int)n, nullptr, rtv, s->p0);
    TRY(spmv(s->p0, nullptr, s->s));
    {
        const double* xs[1] = {s->p0};
        const double* ys[1] = {s->s};
        TRY(launch_dots(a, st, s->part, s->counter, s->dout, 1, xs, ys, nullptr));
    }
    k_init_mu<<<1, 1, 0, st>>>(s->ctrl, s->dout, needs_st ? 1 : 0);
    if (needs_st && (v == CGVK_GV || pipe)) k_scale<<<eg, 256, 0, st>>>((int)n, d, s->s, s->st);
    const double* stv = needs_st && (v == CGVK_GV || pipe) ? s->st : s->s;
    const int st_fly = needs_st && !(v == CGVK_GV || pipe);  // PR/M: s~ = d∘s
    const int expr = s->cfg.nu_expression;
    InitExtras e{};
    auto scalar_dots = [&](bool want_delta) -> int {
        const bool want_dhat = expr == CGVK_NU_EXPANDED;
        const double* xs[3];
        const double* ys[3];
        int dx[3], nd = 0;
        if (want_delta) { xs[nd] = rtv; ys[nd] = s->s; dx[nd] = 0; e.slot[nd++] = SDEL; }
        if (want_dhat) { xs[nd] = stv; ys[nd] = s->r; dx[nd] = st_fly; e.slot[nd++] = SDELH; }
        xs[nd] = stv; ys[nd] = s->s; dx[nd] = st_fly; e.slot[nd++] = SGAM;
        e.nd = nd;
        return launch_dots(a, st, s->part, s->counter, s->dout, nd, xs, ys, dx);
    };
    switch (v) {
        case CGVK_HS:
        case CGVK_CG_CG: break;
        case CGVK_M:
        case CGVK_PR:
            TRY(scalar_dots(v == CGVK_PR || expr != CGVK_NU_MEURANT || s->cfg.track_delta));
            break;
        case CGVK_GV:
            TRY(spmv(rtv, nullptr, s->w));
            TRY(spmv(stv, nullptr, s->u));
            e.spmv = 2;
            break;
        default:  // pipelined PR
            TRY(spmv(rtv, nullptr, s->w));
            if (prec && !s->cfg.recompute_w) k_scale<<<eg, 256, 0, st>>>((int)n, d, s->w, s->wt);
            TRY(spmv(stv, nullptr, s->u));
            e.spmv = 2;
            e.prec = prec ? 2 : 0;  // w~ = M w, u~ = M u
            TRY(scalar_dots(expr != CGVK_NU_MEURANT || s->cfg.track_delta));
            break;
    }
    k_init_extras<<<1, 1, 0, st>>>(s->ctrl, s->dout, e);
    InitVecs iv{};
    iv.after_nu[0] = s->p0;
    iv.after_nu[1] = s->s;
    iv.after_mu[0] = (needs_st && (v == CGVK_GV || pipe)) ? s->st : nullptr;
    iv.after_mu[1] = (v == CGVK_GV || pipe) ? s->w : nullptr;
    iv.after_mu[2] = (v == CGVK_GV || pipe) ? s->u : nullptr;
    iv.after_mu[3] = (pipe && prec && !s->cfg.recompute_w) ? s->wt : nullptr;
    k_init_fixup<<<eg, 256, 0, st>>>((int)n, s->ctrl, iv);
    CK(cudaGetLastError());
    s->mirror = c0;
    s->mirror_fresh = false;  // the status is known once the stream gets there
    return CGVK_OK;
}

void free_solver(cgvk_solver s) {
    if (!s) return;
    if (s->a) cudaSetDevice(s->a->device);
    if (s->stream) cudaStreamSynchronize(s->stream);
    if (s->g8) cudaGraphExecDestroy(s->g8);
    for (double* p : {s->slab, s->wpred, s->rank_tot, s->all_tot, s->sbuf_lo, s->sbuf_hi, s->rbuf_lo, s->rbuf_hi})
        dfree(p);
    if (s->stream && s->owns_stream) cudaStreamDestroy(s->stream);
    delete s;
}

int group_step_all(cgvk_solver s, int n_iters);  // cgvk_group.inc
int group_launches_per_iter(cgvk_solver s);      // cgvk_group.inc

int materialize(cgvk_solver s) {
    TRY(refresh_mirror(s));
    if (!s->mirror.form_pending) return CGVK_OK;
    k_set_limit<<<1, 1, 0, s->stream>>>(s->ctrl, s->mirror.k);
    CK(launch(s, s->k1));
    k_set_limit<<<1, 1, 0, s->stream>>>(s->ctrl, s->k_target);
    CK(cudaGetLastError());
    return refresh_mirror(s);
}

// Device pointer to working vector `which` in the reference's state
// (SolverState fields, inc/variants.hpp:108-111): deferred beta-recurrences
// materialised, tilde vectors the fused schedule recomputes on the fly formed
// into `scratch` (n doubles). CGVK_EINVAL when the variant does not allocate it.
int vector_device(cgvk_solver s, int which, double* scratch, const double** out) {
    const int v = s->cfg.variant;
    const bool pipe = v == CGVK_PIPE_PR || v == CGVK_PIPE_PR_M;
    const bool prec = s->prec;
    const double* src = nullptr;
    const double* scale_src = nullptr;  // out = d∘scale_src
    bool zeros = false;
    TRY(materialize(s));
    const Ctrl& c = s->mirror;
    // initialize() settled the status before resizing the later vectors
    // (src/variants.cpp:383, 389)
    if (c.init_stage == 1 && which != CGVK_VEC_X && which != CGVK_VEC_R && which != CGVK_VEC_R_TILDE)
        return set_err(CGVK_EINVAL, "vector %d was not allocated: initialize() stopped at nu0", which);
    if (c.init_stage == 2 && which != CGVK_VEC_X && which != CGVK_VEC_R && which != CGVK_VEC_R_TILDE &&
        which != CGVK_VEC_P && which != CGVK_VEC_S)
        return set_err(CGVK_EINVAL, "vector %d was not allocated: initialize() stopped at mu0", which);
    switch (which) {
        case CGVK_VEC_X: src = s->x; break;
        // (one-kernel schedules: the current buffer set by ctrl->pcur; w / u / t
        // may hold second buffers of a variant that does not allocate them)
        case CGVK_VEC_R:
            src = ((s->fused == 1 || s->fused == 4) && !prec && c.pcur) ? s->g2
                  : (s->fused == 2 && c.pcur)                          ? s->r2
                                                                       : s->r;
            break;
        case CGVK_VEC_P: src = ((v == CGVK_HS || s->fused == 1) && c.pcur) ? s->p1 : s->p0; break;
        case CGVK_VEC_S:
            src = ((s->fused == 1 || s->fused == 2) && c.pcur) ? s->s2
                  : (s->fused == 4 && !prec && c.pcur)         ? s->a2
                                                               : s->s;
            break;
        case CGVK_VEC_W: src = s->fused == 1 ? nullptr : (s->fused >= 2 && c.pcur) ? s->w2 : s->w; break;
        case CGVK_VEC_U: src = s->fused >= 3 ? (c.pcur ? s->u2 : s->u) : s->fused ? nullptr : s->u; break;
        case CGVK_VEC_T: src = s->fused == 3 ? (c.pcur ? s->t2 : s->t) : s->fused ? nullptr : s->t; break;
        case CGVK_VEC_R_TILDE:
            if (!prec) break;
            if (s->fused == 2) scale_src = c.pcur ? s->r2 : s->r;  // (CgF never stores r~)
            else if (s->rt) src = ((s->fused == 1 || s->fused == 4) && c.pcur) ? s->g2 : s->rt;
            else scale_src = s->r;
            break;
        case CGVK_VEC_S_TILDE:
            if (!prec || v == CGVK_HS || v == CGVK_CG_CG) break;
            if (s->st) src = (s->fused == 4 && c.pcur) ? s->a2 : s->st;
            else scale_src = (s->fused == 1 && c.pcur) ? s->s2 : s->s;
            break;
        case CGVK_VEC_W_TILDE:
            if (!prec || !(v == CGVK_GV || pipe)) break;
            if (v == CGVK_GV) {
                if (c.k == 0) zeros = true;  // resized, never applied before step 1
                else scale_src = (s->fused == 3 && c.pcur) ? s->w2 : s->w;
            } else if (!s->cfg.recompute_w || c.wt_stored) {
                src = s->wt;
            } else {
                scale_src = (s->fused == 4 && c.pcur) ? s->w2 : s->w;
            }
            break;
        case CGVK_VEC_U_TILDE:
            if (!prec || !pipe) break;
            scale_src = (s->fused == 4 && c.pcur) ? s->u2 : s->u;
            break;
        default: break;
    }
    if (!src && !scale_src && !zeros) return set_err(CGVK_EINVAL, "vector %d is not allocated by this variant", which);
    if (zeros) {
        CK(cudaMemsetAsync(scratch, 0, 8 * s->n, s->stream));
        src = scratch;
    } else if (scale_src) {
        k_scale<<<grid_elem(s->n), 256, 0, s->stream>>>((int)s->n, s->a->inv_diag, scale_src, scratch);
        CK(cudaGetLastError());
        src = scratch;
    }
    *out = src;
    return CGVK_OK;
}

}  // namespace

extern "C" {

}  // extern "C"

// Allocate a solver's device state for matrix `a`, choose its kernels; uses
// `stream` when given (a local group shares one), else creates its own.
// allow_fuse: 1 = a single-GPU solver, 2 = a rank of a peer-memory group
// (PrF only), 0 = two kernels per iteration.
int solver_alloc(cgvk_matrix a, const cgvk_variant_config* cfg, int precond, cudaStream_t stream,
                 cgvk_solver* out, int allow_fuse = 0) {
    *out = nullptr;
    if (!a) return set_err(CGVK_EINVAL, "null matrix");
    TRY(cgvk_variant_config_validate(cfg));
    if (precond != CGVK_PRECOND_IDENTITY && precond != CGVK_PRECOND_JACOBI)
        return set_err(CGVK_EINVAL, "unknown preconditioner kind %d", precond);
    CK(cudaSetDevice(a->device));
    if (precond == CGVK_PRECOND_JACOBI) {
        std::lock_guard<std::mutex> lock(a->mu);
        TRY(ensure_jacobi(a));
    }
    auto* s = new cgvk_solver_s;
    s->a = a;
    s->cfg = *cfg;
    s->prec = precond == CGVK_PRECOND_JACOBI;
    s->n = a->n;
    const int v = cfg->variant;
    const bool pipe = v == CGVK_PIPE_PR || v == CGVK_PIPE_PR_M;
    const int64_t n = a->n;
    int rc;
    auto bail = [&](int code) {
        free_solver(s);
        return code;
    };
    s->hist_cap = CGVK_HISTORY_CAP;
    // + halo columns of a rank-local matrix; + 32: bulk copies of the last
    // tile round up to 16 bytes
    const int64_t nv = (a->ncols + 32 + 15) & ~(int64_t)15;
    // One stream-ordered allocation for the solver's vectors and small arrays
    // (each pool allocation is a host round trip: measured 0.17-0.22 ms of a
    // 0.4 ms solver creation on P2D with ~20 separate ones): `want` records a
    // 128-byte-aligned segment, `slab` backs them all.
    struct Seg {
        void** dst;
        size_t doubles;
    };
    std::vector<Seg> segs;
    auto want = [&segs](auto** p, size_t doubles) {
        segs.push_back({reinterpret_cast<void**>(p), (doubles + 15) & ~(size_t)15});
        return 0;
    };
    if ((rc = want(&s->x, nv)) || (rc = want(&s->r, nv)) || (rc = want(&s->p0, nv)) ||
        (rc = want(&s->s, nv)) || (rc = want(&s->b, nv)) || (rc = want(&s->tmp, nv)) ||
        (rc = want(&s->part, 2 * kMaxDots * (size_t)a->gmax + 4)) ||
        (rc = want(&s->hist, s->hist_cap)) ||
        (rc = want(&s->dout, 8)) || (rc = want(&s->counter, 2)) || (rc = want(&s->ctrl, 2 * sizeof(Ctrl) / 8)))
        return bail(rc);
    // PR / M on a problem that fits L2 (CSR engine, chained graphs): one kernel
    // per iteration (PrF); CGVK_FUSE=0 keeps the two-kernel schedule
    // (CGVK_FUSE bit 0: PR / M, bit 1: CG-CG, bit 2: GV, bit 4: pipe-PR; bit 3: GV / pipe-PR at any size)
    const bool small = allow_fuse && a->band_h < 0 && a->l2pol == 3 && use_chain() &&
                       // (the peer form runs 2 CTAs per SM: while every CTA holds one tile — measured
                       // per rank-iteration at P64: 128-tile shards 15.2 -> 14.0 us, 256 tiles 16.9 ->
                       // 13.3, but 512 tiles 16.3 -> 17.0 and 1024 tiles 17.2 -> 19.8)
                       (allow_fuse == 2 ? ((v == CGVK_M || v == CGVK_PR) && a->ntiles <= 2 * a->sms) : a->nranks <= 1);
    const int fuse_env = env_int("CGVK_FUSE", 23);
    const bool one_tile = a->ntiles <= 2 * a->sms || (fuse_env & 8);
    s->fused = !small                                            ? 0
               : ((v == CGVK_M || v == CGVK_PR) && (fuse_env & 1)) ? 1
               : (v == CGVK_CG_CG && (fuse_env & 2))               ? 2
               // (GvF runs 2 CTAs per SM: only while every CTA has one tile — measured
               // P2D 10.7 -> 7.1 us, but P64, 1024 tiles on 222 CTAs, 15.6 -> 18.2 us)
               : (v == CGVK_GV && (fuse_env & 4) && one_tile) ? 3
               // (PprF: the same 2-CTA kernel shape; recompute_w on, as the paper's pipe-PR)
               : (pipe && cfg->recompute_w && (fuse_env & 16) && one_tile) ? 4
                                                                   : 0;
    if (s->fused == 1) {  // second buffers of p, s and r~ (or r)
        if ((rc = want(&s->p1, nv)) || (rc = want(&s->w, nv)) || (rc = want(&s->u, nv))) return bail(rc);
    }
    if (s->fused == 4) {  // second buffers of s~ | s, r~ | r, w and u
        if ((rc = want(&s->b0, nv)) || (rc = want(&s->b1, nv)) || (rc = want(&s->b2, nv)) ||
            (rc = want(&s->p1, nv)))
            return bail(rc);
    }
    if (s->fused == 3) {  // second buffers of w, u and t
        if ((rc = want(&s->b0, nv)) || (rc = want(&s->b1, nv)) || (rc = want(&s->b2, nv))) return bail(rc);
    }
    if (s->fused == 2) {  // second buffers of r, s and w (Params u, t, p1)
        if ((rc = want(&s->u, nv)) || (rc = want(&s->t, nv)) || (rc = want(&s->p1, nv))) return bail(rc);
    }
    if (v == CGVK_HS && (rc = want(&s->p1, nv))) return bail(rc);
    if ((v == CGVK_CG_CG || v == CGVK_GV || pipe) && (rc = want(&s->w, nv))) return bail(rc);
    if ((v == CGVK_GV || pipe) && (rc = want(&s->u, nv))) return bail(rc);
    if (v == CGVK_GV && (rc = want(&s->t, nv))) return bail(rc);
    if (s->prec && (rc = want(&s->rt, nv))) return bail(rc);
    if (s->prec && (v == CGVK_GV || pipe) && (rc = want(&s->st, nv))) return bail(rc);
    if (s->prec && (v == CGVK_GV || pipe) && (rc = want(&s->wt, nv))) return bail(rc);
    {
        size_t total = 0;
        for (const Seg& g : segs) total += g.doubles;
        if ((rc = dalloc(&s->slab, total)) != CGVK_OK) return bail(rc);
        double* at = s->slab;
        for (const Seg& g : segs) {
            *g.dst = at;
            at += g.doubles;
        }
    }
    // the one-kernel schedules' names for their second buffers
    if (s->fused == 1) s->s2 = s->w, s->g2 = s->u;
    if (s->fused == 2) s->r2 = s->u, s->s2 = s->t, s->w2 = s->p1;
    if (s->fused == 3) s->w2 = s->b0, s->u2 = s->b1, s->t2 = s->b2;
    if (s->fused == 4) s->a2 = s->b0, s->g2 = s->b1, s->w2 = s->b2, s->u2 = s->p1;
    if (stream) {
        s->stream = stream;
        s->owns_stream = false;
    } else if (cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking) != cudaSuccess) {
        return bail(set_err(CGVK_ECUDA, "stream create failed"));
    }
    {   // zero everything but the residual history (1 MB, written before it is read): one memset
        size_t lo = 0, hist_at = 0, total = 0;
        for (const Seg& g : segs) {
            if (g.dst == reinterpret_cast<void**>(&s->hist)) hist_at = total;
            total += g.doubles;
        }
        const size_t hist_len = (size_t)(((size_t)s->hist_cap + 15) & ~(size_t)15);
        (void)lo;
        if (cudaMemsetAsync(s->slab, 0, 8 * hist_at, s->stream) != cudaSuccess ||
            (total > hist_at + hist_len &&
             cudaMemsetAsync(s->slab + hist_at + hist_len, 0, 8 * (total - hist_at - hist_len), s->stream) !=
                 cudaSuccess))
            return bail(set_err(CGVK_ECUDA, "memset failed"));
    }
    s->allocated = ref_allocated(v, s->prec);

    Params& P = s->P;
    P = a->base();
    P.d = s->prec ? a->inv_diag : nullptr;
    P.x = s->x;
    P.r = s->r;
    P.p0 = s->p0;
    P.p1 = s->p1;
    P.s = s->s;
    P.w = s->w;
    P.u = s->u;
    P.t = s->t;
    P.rt = s->rt;
    P.st = s->st;
    P.wt = s->wt;
    P.b0 = s->b0;
    P.b1 = s->b1;
    P.b2 = s->b2;
    P.part = s->part;
    P.part_b = s->part + kMaxDots * (size_t)a->gmax;
    P.hist = s->hist;
    P.ctrl = s->ctrl;
    P.ctrl_b = s->ctrl + 1;
    P.nu_expr = cfg->nu_expression;
    P.recompute_nu = cfg->recompute_nu;
    P.recompute_w = cfg->recompute_w;
    P.unsimplified_mu = cfg->unsimplified_mu;
    P.track_delta = cfg->track_delta;
    if ((rc = s->prec ? pick_kernels<true>(a, v, s) : pick_kernels<false>(a, v, s)) != CGVK_OK)
        return bail(rc);
    *out = s;
    return CGVK_OK;
}

extern "C" {

int cgvk_solver_create(cgvk_matrix a, const cgvk_variant_config* cfg, int precond, const double* b,
                       const double* x0, cgvk_solver* out) {
    PhaseTimer pt("solver_create");
    if (!out) return set_err(CGVK_EINVAL, "null output handle");
    *out = nullptr;
    if (!b || !x0) return set_err(CGVK_EINVAL, "right-hand side or initial guess dimension mismatch");
    if (a && a->nranks > 1)
        return set_err(CGVK_EINVAL, "a rank-local matrix needs cgvk_group_create");
    cgvk_solver s = nullptr;
    TRY(solver_alloc(a, cfg, precond, nullptr, &s, /*allow_fuse=*/1));
    int rc;
    auto bail = [&](int code) {
        free_solver(s);
        return code;
    };
    const int64_t n = a->n;
    if (n == 0) {  // r0 is empty: nu0 = 0 = <r,r> -> Converged(ZeroResidual)
        Ctrl c{};
        c.state = ST_CONVERGED;
        c.criterion = CB_ZERO;
        c.stats[STAT_SPMV] = 1;
        c.stats[STAT_PREC] = s->prec;
        c.stats[STAT_RED] = 1;
        c.hist_cap = 0;
        s->mirror = c;
        if (cudaMemcpy(s->ctrl, &c, sizeof(Ctrl), cudaMemcpyHostToDevice) != cudaSuccess)
            return bail(set_err(CGVK_ECUDA, "ctrl upload failed"));
        *out = s;
        return CGVK_OK;
    }
    pt.mark("alloc+kernels");
    if ((rc = solver_init(s, b, x0)) != CGVK_OK) return bail(rc);
    pt.mark("initialize");
    s->gn = graph_iters();
    if ((rc = capture(s, s->gn, &s->g8)) != CGVK_OK) return bail(rc);
    pt.mark("graphs");
    if (env_int("CGVK_SYNC_CREATE", 0) && (rc = refresh_mirror(s)) != CGVK_OK) return bail(rc);
    *out = s;
    return CGVK_OK;
}

int cgvk_solver_destroy(cgvk_solver s) {
    free_solver(s);
    return CGVK_OK;
}

int cgvk_solver_set_tolerance(cgvk_solver s, double rel_tol) {
    if (!s) return set_err(CGVK_EINVAL, "null solver");
    CK(cudaSetDevice(s->a->device));
    if (s->n == 0) return CGVK_OK;
    k_set_tol<<<1, 1, 0, s->stream>>>(s->ctrl, rel_tol);  // stream-ordered, like step()
    CK(cudaGetLastError());
    s->mirror.tol = rel_tol;
    return CGVK_OK;
}

int cgvk_solver_step(cgvk_solver s, int n_iters) {
    if (!s) return set_err(CGVK_EINVAL, "null solver");
    if (n_iters < 0) return set_err(CGVK_EINVAL, "n_iters must be >= 0");
    // a rank of a row-partitioned solve steps every rank this process drives
    if (s->group) return group_step_all(s, n_iters);
    if (s->mirror_fresh && s->mirror.state != ST_RUNNING)
        return set_err(CGVK_ESTATE, "step() on a terminated solver");
    if (n_iters == 0 || s->n == 0) return CGVK_OK;
    CK(cudaSetDevice(s->a->device));
    s->k_target += n_iters;
    k_set_limit<<<1, 1, 0, s->stream>>>(s->ctrl, s->k_target);
    for (int i = 0; i < n_iters / s->gn; ++i) CK(cudaGraphLaunch(s->g8, s->stream));
    TRY(launch_chain(s, n_iters % s->gn));
    CK(cudaGetLastError());
    s->mirror_fresh = false;
    return CGVK_OK;
}

int cgvk_solver_sync(cgvk_solver s) {
    if (!s) return set_err(CGVK_EINVAL, "null solver");
    CK(cudaSetDevice(s->a->device));
    if (s->n == 0) return CGVK_OK;
    return refresh_mirror(s);
}

int cgvk_solver_status(cgvk_solver s, cgvk_solve_status* st, cgvk_scalars* sc, cgvk_stats* stats) {
    if (!s) return set_err(CGVK_EINVAL, "null solver");
    if (!s->mirror_fresh) TRY(cgvk_solver_sync(s));
    const Ctrl& c = s->mirror;
    if (st) {
        st->state = c.state;
        st->breakdown = c.reason;
        st->criterion = c.criterion;
        st->k = c.k;
        // initialize() returns before resizing the later vectors when a check
        // settles the status (src/variants.cpp:383, 389): x r (r~) after the
        // nu0 check, + p s after the mu0 check
        st->allocated_vectors = c.init_stage == 1   ? 2 + s->prec
                                : c.init_stage == 2 ? 4 + s->prec
                                                    : s->allocated;
    }
    if (sc) {
        sc->alpha = c.sc[SA];
        sc->beta = c.sc[SB];
        sc->nu = c.sc[SNU];
        sc->nu_prime = c.sc[SNUP];
        sc->mu = c.sc[SMU];
        sc->delta = c.sc[SDEL];
        sc->delta_hat = c.sc[SDELH];
        sc->gamma = c.sc[SGAM];
        sc->eta = c.sc[SETA];
        sc->rr = c.rr;
    }
    if (stats) {
        stats->spmv_calls = c.stats[STAT_SPMV];
        stats->block_spmv_calls = c.stats[STAT_BLOCK];
        stats->precond_applies = c.stats[STAT_PREC];
        stats->reductions = c.stats[STAT_RED];
    }
    return CGVK_OK;
}

int cgvk_solver_get_vector(cgvk_solver s, int which, double* out) {
    if (!s || !out) return set_err(CGVK_EINVAL, "null argument");
    CK(cudaSetDevice(s->a->device));
    if (s->n == 0) {
        if (which == CGVK_VEC_X || which == CGVK_VEC_R || which == CGVK_VEC_P || which == CGVK_VEC_S)
            return CGVK_OK;
    }
    const double* src = nullptr;
    TRY(vector_device(s, which, s->tmp, &src));
    CK(cudaMemcpyAsync(out, src, 8 * s->n, cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    return CGVK_OK;
}

int cgvk_solver_get_vector_async(cgvk_solver s, int which, double* out) {
    if (!s || !out) return set_err(CGVK_EINVAL, "null argument");
    if (which != CGVK_VEC_X) return set_err(CGVK_EINVAL, "asynchronous download is for x only");
    CK(cudaSetDevice(s->a->device));
    if (s->n == 0) return CGVK_OK;
    // x is never deferred: both kernels of every iteration leave x_k complete
    CK(cudaMemcpyAsync(out, s->x, 8 * s->n, cudaMemcpyDeviceToHost, s->stream));
    s->mirror_fresh = false;
    return CGVK_OK;
}

int cgvk_solver_after(cgvk_solver s, cgvk_solver prev) {
    if (!s || !prev) return set_err(CGVK_EINVAL, "null solver");
    if (s->a->device != prev->a->device) return set_err(CGVK_EINVAL, "solvers on different devices");
    CK(cudaSetDevice(s->a->device));
    if (s->stream == prev->stream) return CGVK_OK;
    cudaEvent_t ev;
    CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    cudaError_t e = cudaEventRecord(ev, prev->stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s->stream, ev, 0);
    cudaEventDestroy(ev);  // released once the wait is resolved
    CK(e);
    return CGVK_OK;
}

int cgvk_solver_true_residual(cgvk_solver s, double* out) {
    if (!s || !out) return set_err(CGVK_EINVAL, "null argument");
    CK(cudaSetDevice(s->a->device));
    if (s->n == 0) {
        *out = 0.0;
        return CGVK_OK;
    }
    Params P = s->a->base();
    if (s->a->spmv_eng) {  // the engines' residual form (built by initialize for a plain matrix)
        Params Q = P;
        Q.w = s->x;
        Q.u = s->b;
        Q.t = s->tmp;
        CK(launch_with(s->stream, s->a->spmv_eng->L[2], Q));
    } else {
        k_spmv<<<s->a->G, kBlock, 0, s->stream>>>(P, s->x, s->b, s->tmp, 0);
    }
    CK(cudaGetLastError());
    const double* xs[1] = {s->tmp};
    double h[1];
    TRY(run_dots(s->a, s->stream, s->part, s->counter, s->dout, 1, xs, xs, nullptr, h));
    *out = std::sqrt(h[0]);
    return CGVK_OK;
}

int cgvk_solver_history(cgvk_solver s, double* out, int cap, int* len) {
    if (!s || !len) return set_err(CGVK_EINVAL, "null argument");
    TRY(cgvk_solver_sync(s));
    int m = s->mirror.k + 1;
    if (m > s->hist_cap) m = s->hist_cap;
    if (s->n == 0) m = 0;
    if (out && cap > 0) {
        const int c = m < cap ? m : cap;
        std::vector<double> h(c);
        if (c) CK(cudaMemcpy(h.data(), s->hist, 8 * c, cudaMemcpyDeviceToHost));
        for (int i = 0; i < c; ++i) out[i] = std::sqrt(h[i]);
    }
    *len = m;
    return CGVK_OK;
}

void* cgvk_solver_stream(cgvk_solver s) { return s ? (void*)s->stream : nullptr; }

int cgvk_solver_launches_per_iter(cgvk_solver s) {
    if (!s) return 0;
    return s->group ? group_launches_per_iter(s) : s->fused ? 1 : 2;
}

long long cgvk_solver_launches(cgvk_solver s, int n_iters) {
    if (!s || n_iters <= 0) return 0;
    if (s->group) return 1 + (long long)group_launches_per_iter(s) * n_iters;
    const long long graphs = n_iters / s->gn + (n_iters % s->gn ? 1 : 0);  // chained runs (one tail each)
    return 1 + (s->fused ? 1LL : 2LL) * n_iters + (use_chain() ? graphs : 0);
}

int cgvk_solver_time_steps(cgvk_solver s, int n_iters, double* ms, int* iters) {
    if (!s || !ms || !iters) return set_err(CGVK_EINVAL, "null argument");
    CK(cudaSetDevice(s->a->device));
    TRY(refresh_mirror(s));
    const int k0 = s->mirror.k;
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, s->stream));
    // a member of an in-process group times the whole group's iterations
    const int rc = s->group ? group_step_all(s, n_iters) : cgvk_solver_step(s, n_iters);
    CK(cudaEventRecord(e1, s->stream));
    CK(cudaEventSynchronize(e1));
    float f = 0.f;
    CK(cudaEventElapsedTime(&f, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    TRY(rc);
    TRY(refresh_mirror(s));
    *ms = f;
    *iters = s->mirror.k - k0;
    return CGVK_OK;
}

int cgvk_solver_profile(cgvk_solver s, int n_iters, double* k1_ms, double* k2_ms, int* iters) {
    if (!s || !k1_ms || !k2_ms || !iters) return set_err(CGVK_EINVAL, "null argument");
    CK(cudaSetDevice(s->a->device));
    TRY(refresh_mirror(s));
    if (s->mirror.state != ST_RUNNING) return set_err(CGVK_ESTATE, "step() on a terminated solver");
    const int k0 = s->mirror.k;
    s->k_target += n_iters;
    k_set_limit<<<1, 1, 0, s->stream>>>(s->ctrl, s->k_target);
    std::vector<cudaEvent_t> ev(3 * (size_t)n_iters);
    for (auto& e : ev) CK(cudaEventCreate(&e));
    for (int i = 0; i < n_iters; ++i) {
        CK(cudaEventRecord(ev[3 * i], s->stream));
        CK(launch(s, s->k1));
        CK(cudaEventRecord(ev[3 * i + 1], s->stream));
        if (!s->fused) CK(launch(s, s->k2));  // (one kernel per iteration: k2_ms = 0)
        CK(cudaEventRecord(ev[3 * i + 2], s->stream));
    }
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(s->stream));
    double a = 0.0, b = 0.0;
    for (int i = 0; i < n_iters; ++i) {
        float f1 = 0.f, f2 = 0.f;
        CK(cudaEventElapsedTime(&f1, ev[3 * i], ev[3 * i + 1]));
        CK(cudaEventElapsedTime(&f2, ev[3 * i + 1], ev[3 * i + 2]));
        a += f1;
        b += f2;
    }
    for (auto& e : ev) cudaEventDestroy(e);
    TRY(refresh_mirror(s));
    *k1_ms = a;
    *k2_ms = b;
    *iters = s->mirror.k - k0;
    return CGVK_OK;
}

int cgvk_solve(cgvk_matrix a, const cgvk_variant_config* cfg, int precond, const double* b,
               const double* x0, int max_iter, double rel_tol, double* x_out, cgvk_solve_status* st,
               cgvk_scalars* sc) {
    if (max_iter < 0) return set_err(CGVK_EINVAL, "max_iter must be >= 0");
    cgvk_solver s = nullptr;
    TRY(cgvk_solver_create(a, cfg, precond, b, x0, &s));
    int rc = CGVK_OK;
    if (rel_tol > 0.0) rc = cgvk_solver_set_tolerance(s, rel_tol);
    // one host sync for the whole solve: iterations after a terminal status
    // (also one settled by initialize) are device-side no-ops
    if (rc == CGVK_OK) rc = cgvk_solver_step(s, max_iter);
    if (rc == CGVK_OK && x_out) rc = cgvk_solver_get_vector_async(s, CGVK_VEC_X, x_out);
    if (rc == CGVK_OK) rc = cgvk_solver_sync(s);
    cgvk_solve_status tmp{};
    if (rc == CGVK_OK) rc = cgvk_solver_status(s, &tmp, sc, nullptr);
    // run(): a budget exhausted while running reports MaxIterations
    // (src/runner.cpp:138)
    if (rc == CGVK_OK && tmp.state == CGVK_RUNNING) tmp.state = CGVK_MAX_ITERATIONS;
    if (st) *st = tmp;
    cgvk_solver_destroy(s);
    return rc;
}

}  // extern "C"

#include "cgvk_group.inc"
#include "cgvk_run.inc"
