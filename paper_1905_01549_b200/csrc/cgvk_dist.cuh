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
    if (threadIdx.x != 0) return;
    pdl_wait();
    Op op;
    if (!op.enter(P)) return;  // nothing was reduced (or it already finished locally)
    if (op.sync() != 2) return;
    double tot[Op::ND > 0 ? Op::ND : 1];
#pragma unroll
    for (int d = 0; d < Op::ND; ++d) tot[d] = 0.0;
    for (int r = 0; r < nranks; ++r) {
#pragma unroll
        for (int d = 0; d < Op::ND; ++d) tot[d] = ADD(tot[d], all_tot[r * kMaxDots + d]);
    }
    op.finish(P, P.ctrl, tot);
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
