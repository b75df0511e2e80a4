// Row-partitioned (multi-rank) pieces of the device path: the rank-ordered
// finalisation of a reduction and the halo pack/unpack kernels.
//
// A rank owns rows [lo, hi) of A in local numbering [own | lower halo | upper
// halo]; the SpMV kernels are the single-GPU ones, gathering from the halo
// region. A reducing kernel in a rank stops at its rank-local total
// (Params::rank_tot); once all ranks' totals are exchanged, k_finalize sums
// them in rank order from 0.0 — the oracle's ORC_DOT_PART order — and runs
// the Op's scalar tail, so every rank holds bit-identical scalars and status.
#pragma once

#include "cgvk_device.cuh"

namespace cgvk {

template <class Op>
__global__ void k_finalize(Params P, const double* __restrict__ all_tot, int nranks) {
    // one warp: the control block and the rank totals come in with one load
    // each per lane; enter/finish run on the shared copy; only the words
    // finish changed are written back (K2 of an overlapped GV / pipe-PR step
    // may be ending concurrently and writes its own, disjoint field)
    constexpr int kWords = sizeof(Ctrl) / 4;
    __shared__ __align__(16) Ctrl cs;
    __shared__ double at[64 * kMaxDots];
    const int t = threadIdx.x;
    pdl_wait();
    unsigned int* cw = reinterpret_cast<unsigned int*>(&cs);
    unsigned int* gw = reinterpret_cast<unsigned int*>(P.ctrl);
    unsigned int orig[(kWords + 31) / 32];
#pragma unroll
    for (int u = 0; u < (kWords + 31) / 32; ++u) {
        const int q = t + 32 * u;
        if (q < kWords) cw[q] = orig[u] = __ldcg(gw + q);
    }
    for (int q = t; q < nranks * kMaxDots; q += 32) at[q] = __ldcg(all_tot + q);
    __syncwarp();
    if (t == 0) {
        Params Q = P;
        Q.ctrl = &cs;
        Op op;
        if (op.enter(Q) && op.sync() == 2) {  // else nothing was reduced (or it finished locally)
            double tot[Op::ND > 0 ? Op::ND : 1];
#pragma unroll
            for (int d = 0; d < Op::ND; ++d) tot[d] = 0.0;
            for (int r = 0; r < nranks; ++r) {
#pragma unroll
                for (int d = 0; d < Op::ND; ++d) tot[d] = ADD(tot[d], at[r * kMaxDots + d]);
            }
            op.finish(Q, &cs, tot);
        }
    }
    __syncwarp();
#pragma unroll
    for (int u = 0; u < (kWords + 31) / 32; ++u) {
        const int q = t + 32 * u;
        if (q < kWords && cw[q] != orig[u]) gw[q] = cw[q];
    }
}

// The vector a halo exchange moves: `a`, or HS's current p (a/b by ctrl->pcur).
struct VecSel {
    double* a;
    double* b;
    const Ctrl* ctrl;
    __device__ __forceinline__ double* get() const { return (b && ctrl->pcur) ? b : a; }
};

// out[q] = v[idx[q]] (the rows a neighbour references)
__global__ void k_halo_pack(VecSel sel, const int* __restrict__ idx, int cnt, double* __restrict__ out) {
    const double* v = sel.get();
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < cnt; q += gridDim.x * blockDim.x)
        out[q] = v[idx[q]];
}

// v[dst0 + q] = in[q] (a neighbour's rows into this rank's halo region)
__global__ void k_halo_unpack(VecSel sel, int dst0, const double* __restrict__ in, int cnt) {
    double* v = sel.get();
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < cnt; q += gridDim.x * blockDim.x)
        v[dst0 + q] = in[q];
}

// In-process transport: every rank's all_tot[r] = rank r's rank_tot.
struct TotTable {
    const double* src[64];
    double* dst[64];
};

__global__ void k_gather_tot(TotTable T, int nranks) {
    const int q = blockIdx.x, r = threadIdx.x / kMaxDots, d = threadIdx.x % kMaxDots;
    if (q < nranks && r < nranks) T.dst[q][r * kMaxDots + d] = T.src[r][d];
}

}  // namespace cgvk
