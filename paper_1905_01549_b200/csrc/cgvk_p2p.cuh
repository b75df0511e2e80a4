// Peer-memory exchange of a row-partitioned solve (north star
// (3)): NVLink P2P stores from the producing kernel and stamped reads in the
// consuming kernel — no NCCL call, no exchange or finalize launch, and no
// memory fence inside the iteration.
//
// A rank's chained kernels (cgvk_stream.cuh, CSR engine, z-slab partitions:
// a rank sends a row prefix to its lower and a row suffix to its upper
// neighbour) carry a kernel sequence number `hseq` in the control block —
// +1 per K1 / K2, identical on every rank because every rank runs the same
// schedule on bit-identical scalars. Everything exchanged travels as "LL"
// words (NCCL's low-latency idea): 32 data bits + the 32-bit stamp (the
// producer's hseq) in one 8-byte store, so a reader that sees the stamp it
// expects in a word has that word's data — no fence on either side.
//
//  * halo: a kernel that updates a halo-exchanged vector pushes its boundary
//    rows into the neighbour's receive buffer (two words per double, parity
//    buffer (stamp >> 1) & 1). The consumer's SpMV gathers a halo column
//    (j >= hbase) from that buffer, spinning until the stamp is the one it
//    expects (its own hseq minus the slot's distance). Only boundary rows
//    read the halo, so the interior SpMV never waits: it overlaps the
//    exchange by construction.
//  * rank totals: the reducing kernel's last CTA writes its rank-local total
//    into table (stamp & 3) of every rank; the successor's prologue (warp 0)
//    polls the words and folds the totals in rank order from 0.0 — the
//    oracle's ORC_DOT_PART order, so every rank runs the scalar tail on
//    identical bits. GV's and pipe-PR's K1 reductions are not waited for by
//    K2 (their SpMV needs no scalar): K2 takes the go-ahead (dist_mark) and
//    the NEXT K1 folds them — Table 1's max(C_gr, T_mv + C_mv).
//  * buffer reuse: a producer writes a halo buffer parity again two
//    iterations later, after folding a reduction that the consumer published
//    only after it had finished reading it (every variant reduces at least
//    once per iteration, in a kernel after the consumer in stream order), so
//    no ack or back-pressure flag is needed.
//
// Every wait is bounded: a wait that gives up sets pp.err (the host reports
// CGVK_ECUDA) and the kernel proceeds, so a broken peer never hangs the GPU.
#pragma once

#include "cgvk_device.cuh"

namespace cgvk {

// Memory scope of the exchange: system (peers on other GPUs over NVLink). An
// A/B build may use -DCGVK_P2P_SCOPE=gpu for in-process ranks on one device.
#ifndef CGVK_P2P_SCOPE
#define CGVK_P2P_SCOPE sys
#endif
#define CGVK_STR2(x) #x
#define CGVK_STR(x) CGVK_STR2(x)
#define CGVK_SCOPE_S CGVK_STR(CGVK_P2P_SCOPE)

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed." CGVK_SCOPE_S ".global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void ld_relaxed_v2u64(const unsigned long long* p, unsigned long long& a,
                                                 unsigned long long& b) {
    asm volatile("ld.relaxed." CGVK_SCOPE_S ".global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}

// A/B of the LL store form (CGVK_P2P_ST: 0 relaxed at the exchange scope,
// 1 volatile, 2 weak)
#ifndef CGVK_P2P_ST
#define CGVK_P2P_ST 0
#endif
__device__ __forceinline__ void st_relaxed_v2u64(unsigned long long* p, unsigned long long a, unsigned long long b) {
#if CGVK_P2P_ST == 1
    asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
#elif CGVK_P2P_ST == 2
    asm volatile("st.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
#else
    asm volatile("st.relaxed." CGVK_SCOPE_S ".global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
#endif
}

constexpr long long kP2pSpinNs = 2000000000ll;  // give up after ~2 s

__device__ __forceinline__ long long gtimer_ns() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// LL words: stamp in the high half, 32 data bits in the low half.
__device__ __forceinline__ unsigned long long ll_word(unsigned int stamp, unsigned int data) {
    return ((unsigned long long)stamp << 32) | data;
}

// ------------------------------------------------------------ rank totals
// Table of rank q: [kP2pTotSlots][kP2pRanks][kLLWords] words: the totals,
// then (latency injection only) the publication time.
constexpr int kLLTime = 2 * kMaxDots;
constexpr int kLLWords = kLLTime + 2;

__device__ __forceinline__ unsigned long long* ll_table(double* base) {
    return reinterpret_cast<unsigned long long*>(base);
}

// Warp 0 (all lanes): the totals stamped `stamp`, summed in rank order from
// 0.0 into lane 0's tot[]. scratch: >= kP2pRanks * kLLWords 32-bit words of
// shared memory.
template <int ND>
__device__ __noinline__ void p2p_fold_totals(const PeerPlan* P2, unsigned int stamp, double* tot,
                                             unsigned int* scratch) {
    const PeerPlan& pp = *P2;
    const int lane = threadIdx.x & 31;
    // the plan's fields in one round of independent loads (lane r: rank r's
    // table pointer; ours is picked by a shuffle)
    const int nranks = __ldg(&pp.nranks), rank = __ldg(&pp.rank);
    const long long delay = __ldg(&pp.delay_ns);
    const unsigned long long mytab = lane < kP2pRanks ? __ldg((const unsigned long long*)&pp.xtot_peer[lane]) : 0ull;
    const unsigned long long* tab = ll_table((double*)__shfl_sync(0xffffffffu, mytab, rank)) +
                                    (size_t)(stamp & (kP2pTotSlots - 1)) * kP2pRanks * kLLWords;
    const int nw = nranks * kLLWords;
    const bool timed = delay > 0;
    long long t0 = 0;
    for (int spin = 0;; ++spin) {
        bool ok = true;
        for (int q = lane; q < nw; q += 32) {
            const int wi = q % kLLWords;
            if (wi >= 2 * ND && (wi < kLLTime || !timed)) continue;
            const unsigned long long w = ld_relaxed_u64(tab + q);
            if ((unsigned int)(w >> 32) == stamp) scratch[q] = (unsigned int)w;
            else ok = false;
        }
        if (__all_sync(0xffffffffu, ok)) break;
        if (spin == 0) t0 = gtimer_ns();
        else if ((spin & 255) == 0 && gtimer_ns() - t0 > kP2pSpinNs) {
            if (lane == 0) atomicExch(P2->err, 1u);
            break;
        }
    }
    __syncwarp();
    if (timed && lane == 0) {  // an injected link latency: arrival = publication + delay
        long long tmax = 0;
        for (int r = 0; r < nranks; ++r) {
            const unsigned int* w = scratch + r * kLLWords + kLLTime;
            const long long tp = (long long)(((unsigned long long)w[1] << 32) | w[0]);
            tmax = tp > tmax ? tp : tmax;
        }
        const long long t1 = gtimer_ns();
        while (gtimer_ns() < tmax + delay) {
            if (gtimer_ns() - t1 > kP2pSpinNs) {  // bounded like every wait
                atomicExch(P2->err, 1u);
                break;
            }
        }
    }
    __syncwarp();
    if (lane == 0) {
#pragma unroll
        for (int d = 0; d < kMaxDots; ++d) tot[d] = 0.0;
        for (int r = 0; r < nranks; ++r) {
#pragma unroll
            for (int d = 0; d < ND; ++d) {
                const unsigned int* w = scratch + r * kLLWords + 2 * d;
                tot[d] = ADD(tot[d], __hiloint2double((int)w[1], (int)w[0]));
            }
        }
    }
    __syncwarp();
}

// One thread (the reducing kernel's last CTA): this rank's total into every
// rank's table (stamp & 3).
template <int ND>
__device__ __noinline__ void p2p_publish_totals(const PeerPlan* P2, unsigned int stamp, const double* tot) {
    const PeerPlan& pp = *P2;
    // every plan field in one round of independent loads (a chain of
    // dependent loads here sits on the critical path of the kernel's end)
    const int nranks = __ldg(&pp.nranks), rank = __ldg(&pp.rank);
    const long long delay = __ldg(&pp.delay_ns);
    unsigned long long ptab[kP2pRanks];
#pragma unroll
    for (int r = 0; r < kP2pRanks; ++r) ptab[r] = __ldg((const unsigned long long*)&pp.xtot_peer[r]);
    const size_t off = ((size_t)(stamp & (kP2pTotSlots - 1)) * kP2pRanks + rank) * kLLWords;
    const unsigned long long tp = delay > 0 ? (unsigned long long)gtimer_ns() : 0ull;
#pragma unroll
    for (int r = 0; r < kP2pRanks; ++r) {
        if (r >= nranks) break;
        unsigned long long* dst = ll_table((double*)ptab[r]) + off;
#pragma unroll
        for (int d = 0; d < ND; ++d)
            st_relaxed_v2u64(dst + 2 * d, ll_word(stamp, (unsigned int)__double2loint(tot[d])),
                             ll_word(stamp, (unsigned int)__double2hiint(tot[d])));
        if (delay > 0)
            st_relaxed_v2u64(dst + kLLTime, ll_word(stamp, (unsigned int)tp), ll_word(stamp, (unsigned int)(tp >> 32)));
    }
}

// ------------------------------------------------------------------- halo

__device__ __forceinline__ int ll_parity(unsigned int stamp) { return (stamp >> 1) & 1; }

// physical slot of HS's p_old (the other p buffer is p_new)
__device__ __forceinline__ int p2p_pold(int pcur) { return pcur ? 2 : 1; }

// A launch's push mask: physical slots, kPushPnew = HS's p_new (by pcur),
// kPushFused = the buffer set a one-kernel iteration (PrF: slots p0 p1 s s2
// g g2, sets {0, 2, 4} / {1, 3, 5}) writes — the other one than ctrl->pcur
// names. A launch that does not step pushes the set its successor will read
// (the current one), p2p_idle_mask.
constexpr unsigned int kPushPnew = 1u << 8;
constexpr unsigned int kPushFused = 1u << 9;
__device__ __forceinline__ unsigned int p2p_push_mask(unsigned int m, int pcur) {
    if (m & kPushPnew) m = (m & ~kPushPnew) | (1u << (3 - p2p_pold(pcur)));
    if (m & kPushFused) m = pcur ? 0x15u : 0x2au;
    return m;
}
__device__ __forceinline__ unsigned int p2p_idle_mask(unsigned int m, int pcur) {
    if (m & kPushPnew) return 6u;  // HS: both p buffers (the next p_old is this kernel's p_old)
    if (m & kPushFused) return pcur ? 0x2au : 0x15u;
    return m;
}

// The thread's row i of every vector in `mask` (physical slots) into the
// neighbours' receive buffers, stamped h — the value the thread itself just
// stored (re-read from L2). Rows outside the send prefix / suffix: nothing.
__device__ __forceinline__ const void* ldg_ptr(const void* const* p) {
    return (const void*)__ldg((const unsigned long long*)p);
}

__device__ __noinline__ void p2p_push_row(const PeerPlan* P2, unsigned int mask, int i, int n, unsigned int h) {
    const PeerPlan& pp = *P2;
    // plan fields through the read-only path, all issued before the stores
    // (plain loads would be re-issued after every store: the compiler cannot
    // rule out that a remote store aliases the plan)
    const int nlo = __ldg(&pp.nlo), hi0 = __ldg(&pp.hi0);
    const bool lo = i < nlo, hi = i >= hi0 && i < n;
    if (!lo && !hi) return;
    const int lo_stride = __ldg(&pp.lo_stride), lo_off = __ldg(&pp.lo_off), hi_stride = __ldg(&pp.hi_stride);
    const int par = ll_parity(h);
#pragma unroll
    for (int q = 0; q < kP2pSlots; ++q) {
        if (!((mask >> q) & 1)) continue;
        const double* hv = (const double*)ldg_ptr((const void* const*)&pp.hv[q]);
        auto* rlo = (unsigned long long*)ldg_ptr((const void* const*)&pp.rx_lo[q]);
        auto* rhi = (unsigned long long*)ldg_ptr((const void* const*)&pp.rx_hi[q]);
        const double v = __ldcg(hv + i);
        const unsigned long long w0 = ll_word(h, (unsigned int)__double2loint(v));
        const unsigned long long w1 = ll_word(h, (unsigned int)__double2hiint(v));
        if (lo && rlo) st_relaxed_v2u64(rlo + 2 * ((size_t)par * lo_stride + lo_off + i), w0, w1);
        if (hi && rhi) st_relaxed_v2u64(rhi + 2 * ((size_t)par * hi_stride + (i - hi0)), w0, w1);
    }
}

// Halo entry e of vector g (one of pp.hv) as this kernel (sequence number h)
// expects it: spin until both words carry the stamp, then store the double
// into g's halo region (the row's gathers read it back through L2).
__device__ __forceinline__ void p2p_fetch(const PeerPlan& pp, const double* g, int hb, int e, unsigned int h,
                                          int pcur) {
    int q = 0;
    while (q < kP2pSlots - 1 && ldg_ptr((const void* const*)&pp.hv[q]) != (const void*)g) ++q;
    const unsigned int want = h - ((__ldg(&pp.psel) && q == p2p_pold(pcur)) ? 2u : 1u);
    const auto* rx = (const unsigned long long*)ldg_ptr((const void* const*)&pp.rx[q]);
    const unsigned long long* w = rx + 2 * ((size_t)ll_parity(want) * __ldg(&pp.rx_stride) + e);
    long long t0 = 0;
    for (int spin = 0;; ++spin) {
        unsigned long long a, b;
        ld_relaxed_v2u64(w, a, b);
        if ((unsigned int)(a >> 32) == want && (unsigned int)(b >> 32) == want) {
            const_cast<double*>(g)[hb + e] = __hiloint2double((int)(unsigned int)b, (int)(unsigned int)a);
            return;
        }
        if (spin == 0) t0 = gtimer_ns();
        else if ((spin & 255) == 0 && gtimer_ns() - t0 > kP2pSpinNs) {
            atomicExch(pp.err, 1u);
            return;
        }
    }
}

// A boundary row's halo entries (columns >= hb) of the gathered sources g0
// (and g1), fetched before the row is computed. ci: the row's columns (stage
// or global), len entries.
__device__ __noinline__ void p2p_unpack_row(const PeerPlan* P2, const int* ci, int len, int hb, const double* g0,
                                            const double* g1, unsigned int h, int pcur) {
    const PeerPlan& pp = *P2;
    for (int k = 0; k < len; ++k) {
        const int c = ci[k];
        if (c < hb) continue;
        if (g0) p2p_fetch(pp, g0, hb, c - hb, h, pcur);
        if (g1) p2p_fetch(pp, g1, hb, c - hb, h, pcur);
    }
}

// The same for a one-kernel iteration (PrF): three exchanged sources, their
// physical slots known from ctrl->pcur (no pointer search), pushed by the
// previous launch (stamp h - 1); the three entries of a halo column are
// polled together, so a boundary row costs one peer round trip per halo
// column, not three chains of dependent plan loads.
__device__ __noinline__ void p2p_unpack_row3(const PeerPlan* P2, const int* ci, int len, int hb, int pcur,
                                             const double* g0, const double* g1, const double* g2, unsigned int h) {
    const PeerPlan& pp = *P2;
    const unsigned int want = h - 1u;
    const int b = pcur ? 1 : 0;  // slots: p0 p1 | s s2 | g g2
    const auto* r0 = (const unsigned long long*)ldg_ptr((const void* const*)&pp.rx[0 + b]);
    const auto* r1 = (const unsigned long long*)ldg_ptr((const void* const*)&pp.rx[2 + b]);
    const auto* r2 = (const unsigned long long*)ldg_ptr((const void* const*)&pp.rx[4 + b]);
    const size_t base = (size_t)ll_parity(want) * __ldg(&pp.rx_stride);
    for (int k = 0; k < len; ++k) {
        const int c = ci[k];
        if (c < hb) continue;
        const size_t e = 2 * (base + (size_t)(c - hb));
        long long t0 = 0;
        for (int spin = 0;; ++spin) {
            unsigned long long a0, b0, a1, b1, a2, b2;
            ld_relaxed_v2u64(r0 + e, a0, b0);
            ld_relaxed_v2u64(r1 + e, a1, b1);
            ld_relaxed_v2u64(r2 + e, a2, b2);
            const bool ok = (unsigned int)(a0 >> 32) == want && (unsigned int)(b0 >> 32) == want &&
                            (unsigned int)(a1 >> 32) == want && (unsigned int)(b1 >> 32) == want &&
                            (unsigned int)(a2 >> 32) == want && (unsigned int)(b2 >> 32) == want;
            if (ok) {
                const_cast<double*>(g0)[c] = __hiloint2double((int)(unsigned int)b0, (int)(unsigned int)a0);
                const_cast<double*>(g1)[c] = __hiloint2double((int)(unsigned int)b1, (int)(unsigned int)a1);
                const_cast<double*>(g2)[c] = __hiloint2double((int)(unsigned int)b2, (int)(unsigned int)a2);
                break;
            }
            if (spin == 0) t0 = gtimer_ns();
            else if ((spin & 255) == 0 && gtimer_ns() - t0 > kP2pSpinNs) {
                atomicExch(pp.err, 1u);
                break;
            }
        }
    }
}

}  // namespace cgvk
