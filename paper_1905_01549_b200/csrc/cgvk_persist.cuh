// Persistent iteration kernel: K1 and K2 of every iteration in ONE
// cooperative launch (all CTAs co-resident), the phases separated by a grid
// barrier whose last arriving CTA folds the phase's dot partials and runs the
// scalar tail — the same canonical reduction and the same Op code as the
// two-kernel graph path, so the bits are identical. It removes the per-kernel
// launch, pipeline ramp and drain (~5-10 us per kernel), which dominates the
// latency-bound configurations (P64, P2D) and costs a few % on large ones.
//
// One TMA ring serves both phases: its stage layout is the union of the two
// Ops' (CSR region + max(NV1, NV2) vector slots) and the producer and the
// consumers keep one running stage counter across phases.
#pragma once

#include "cgvk_stream.cuh"

namespace cgvk {

struct PersistCfg {
    StageCfg S;  // union stage layout
};

// Producer side of one phase (lane 0 of the producer warp).
template <class Op>
__device__ __forceinline__ void persist_produce(const Params& P, const StageCfg& S, PipeHeader* H,
                                                unsigned char* stages, const Op& op, int& j, uint64_t pol) {
    const int Gv = S.gvirt, Gp = gridDim.x, ntiles = P.ntiles, NS = S.nstage;
    const double* vp[kMaxVec];
#pragma unroll
    for (int v = 0; v < Op::NV; ++v) vp[v] = op.vec(P, v);
    const uint64_t vpol = P.l2pol == 0 ? pol : 0;
    // generic-proxy writes of the previous phase (other CTAs) -> async-proxy reads
    asm volatile("fence.proxy.async.global;" ::: "memory");
    CGVK_FOR_VB(vb, P.order, blockIdx.x, Gv, Gp) {
        CGVK_FOR_TILE(tile, P.order, vb, ntiles, Gv) {
            const int slot = j % NS;
            if (j >= NS) mbar_wait(&H->empty[slot], ((j / NS) - 1) & 1);
            StageView V = stage_view(stages, S, slot);
            const int r0 = tile * kBlock;
            const int rows = min(kBlock, P.n - r0);
            if (Op::CSR) stage_csr(P, S, H, stages, slot, tile, pol, false);
            const uint32_t vec_bytes = (rows * 8 + 15) & ~15;
            uint32_t bytes = 0;
#pragma unroll
            for (int v = 0; v < Op::NV; ++v)
                if (vp[v]) bytes += vec_bytes;
            mbar_expect_tx(&H->full[slot], bytes);
#pragma unroll
            for (int v = 0; v < Op::NV; ++v)
                if (vp[v]) bulk_g2s(V.vec + v * kBlock, vp[v] + r0, vec_bytes, &H->full[slot], vpol);
            ++j;
        }
    }
}

// Consumer side of one phase (the 8 consumer warps): rows, per-virtual-CTA
// canonical trees, partials.
template <class Op>
__device__ __forceinline__ void persist_consume(const Params& P, const StageCfg& S, PipeHeader* H,
                                                unsigned char* stages, const Op& op, int& j) {
    const int Gv = S.gvirt, Gp = gridDim.x, ntiles = P.ntiles, NS = S.nstage;
    const int t = threadIdx.x;
    double acc[Op::ND > 0 ? Op::ND : 1];
    CGVK_FOR_VB(vb, P.order, blockIdx.x, Gv, Gp) {
#pragma unroll
        for (int d = 0; d < Op::ND; ++d) acc[d] = 0.0;
        CGVK_FOR_TILE(tile, P.order, vb, ntiles, Gv) {
            const int jj = j++;
            const int slot = jj % NS;
            mbar_wait(&H->full[slot], (jj / NS) & 1);
            StageView V = stage_view(stages, S, slot);
            const int i = tile * kBlock + t;
            if (i < P.n) {
                RowRef R{nullptr, nullptr, 0};
                if (Op::CSR) {
                    const int b = V.rp[t];
                    R.len = V.rp[t + 1] - b;
                    if (H->direct[slot]) {
                        R.va = P.va + b;
                        R.ci = P.ci + b;
                    } else {
                        R.va = V.va + (b - H->k0a[slot]);
                        R.ci = V.ci + (b - H->k0c[slot]);
                    }
                }
                op.row(P, i, StagedIn{V.vec + t}, R, acc);
            }
            __syncwarp();
            if ((t & 31) == 0) mbar_arrive(&H->empty[slot]);
        }
        if constexpr (Op::ND > 0) {
            if (op.sync() != 2) continue;
            cta_tree_c<Op::ND>(acc, H->red);
            if (t == 0) {
#pragma unroll
                for (int d = 0; d < Op::ND; ++d) P.part[d * Gv + vb] = acc[d];
            }
        }
    }
}

// Grid barrier; the last CTA to arrive folds the partials and runs
// op.finish() before releasing the others. Every thread of the block calls it.
template <class Op>
__device__ __forceinline__ void persist_barrier(const Params& P, const StageCfg& S, PipeHeader* H,
                                                const Op& op, bool active) {
    Ctrl* c = P.ctrl;
    __shared__ unsigned int s_gen;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        s_gen = *reinterpret_cast<volatile unsigned int*>(&c->bar_gen);
        const unsigned int prev = atomicAdd(&c->bar_count, 1u);
        H->last_flag = prev == gridDim.x - 1;
    }
    __syncthreads();
    if (H->last_flag) {
        __threadfence();
        const int mode = active ? op.sync() : 0;
        if (mode > 0 && threadIdx.x < kConsumers) {
            double tot[Op::ND > 0 ? Op::ND : 1];
#pragma unroll
            for (int d = 0; d < Op::ND; ++d) tot[d] = 0.0;
            if constexpr (Op::ND > 0) {
                if (mode == 2) {
                    fold_partials<Op::ND>(P.part, S.gvirt, threadIdx.x, tot);
                    cta_tree_c<Op::ND>(tot, H->red);
                }
            }
            if (threadIdx.x == 0) op.finish(P, c, tot);
        }
        if (threadIdx.x == 0) {
            c->bar_count = 0u;
            __threadfence();
            atomicAdd(&c->bar_gen, 1u);
        }
    } else if (threadIdx.x == 0) {
        while (*reinterpret_cast<volatile unsigned int*>(&c->bar_gen) == s_gen) __nanosleep(64);
        __threadfence();  // acquire; also invalidates this SM's L1 (stale gathers)
    }
    __syncthreads();
}

template <class Op1, class Op2>
__global__ void __launch_bounds__(kThreads, 2) k_persist(Params P, StageCfg S) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    PipeHeader* H = reinterpret_cast<PipeHeader*>(smem_raw);
    unsigned char* stages = smem_raw + ((sizeof(PipeHeader) + 127) / 128) * 128;
    const int NS = S.nstage;
    const bool producer = threadIdx.x == kConsumers;
    const bool consumer = threadIdx.x < kConsumers;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(&H->full[s], 1);
            mbar_init(&H->empty[s], kWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const uint64_t pol = P.l2pol < 2 ? evict_first_policy() : 0;
    int j = 0;  // running stage counter, shared by both phases
    for (;;) {
        {
            Op1 op;
            const bool act = op.enter(P);
            if (act) {
                if (producer) persist_produce(P, S, H, stages, op, j, pol);
                else if (consumer) persist_consume(P, S, H, stages, op, j);
            }
            persist_barrier(P, S, H, op, act);
        }
        {
            Op2 op;
            const bool act = op.enter(P);
            if (act) {
                if (producer) persist_produce(P, S, H, stages, op, j, pol);
                else if (consumer) persist_consume(P, S, H, stages, op, j);
            }
            persist_barrier(P, S, H, op, act);
        }
        if (!step_wanted(P.ctrl)) break;  // uniform: ctrl is stable until the next barrier
    }
}

}  // namespace cgvk
