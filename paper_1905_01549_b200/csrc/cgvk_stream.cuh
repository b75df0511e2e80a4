// The TMA-staged tile pipeline every hot kernel runs on (sm_100a).
//
// A CTA = 8 consumer warps (one row per thread, kBlock = 256 rows per tile)
// + 1 producer warp. The producer streams, per tile, the row_ptr slice, the
// CSR values and column indices of the tile's rows, and each per-row input
// vector the kernel needs, into a ring of shared-memory stages with 1D bulk
// async copies (cp.async.bulk ... mbarrier::complete_tx, "UBLKCP" in SASS),
// NSTAGE tiles ahead. Consumers wait on the stage's full barrier, compute
// their row (the SpMV row product from shared memory, the x gathers through
// L1/L2), store outputs straight to global, fold the dot products, and
// release the stage on its empty barrier. Only the gathered SpMV operand is
// read with ordinary loads.
//
// Reduction order is the canonical one of cgvk_device.cuh, expressed on
// "virtual CTAs": virtual CTA vb (0 <= vb < Gv = min(gmax, ntiles)) owns
// tiles vb, vb+Gv, ... (order 0; order 1: a contiguous run of tiles); a
// physical CTA p runs virtual CTAs p, p+Gp, ... one after the other (Gp =
// resident CTAs), so the result bits do not depend on how many CTAs fit on
// the chip.
//
// The band engine (cgvk_band.cuh) replaces this kernel's SpMV form for
// narrow-band long-row matrices.
#pragma once

#include "cgvk_device.cuh"
#include "cgvk_p2p.cuh"

#include <type_traits>

// Occupancy target of the SpMV kernels (register budget via __launch_bounds__).
// Measured (profiles/r01): 3 resident CTAs per SM for the SpMV kernels (regs
// <= 75, two ring stages) beats 2 CTAs with 3 stages by 5-10 % per kernel.
#ifndef CGVK_SPMV_MIN_CTAS
#define CGVK_SPMV_MIN_CTAS 3
#endif

namespace cgvk {

constexpr int kConsumers = kBlock;           // 8 warps, one row each
constexpr int kThreads = kBlock + 32;        // + producer warp
constexpr int kMaxStages = 8;
constexpr int kRpInts = kBlock + 4;          // row_ptr slice (257 used), padded to 16 B
constexpr int kMaxVec = 12;

// Optional Op hook for row-partitioned solves: `void dist_mark(const Params&,
// Ctrl*) const`, run by the reducing kernel's last CTA when it stops at its
// rank-local total — the control state the NEXT kernel needs before the
// exchanged reduction is finalised (GV / pipe-PR overlap that finalisation
// with their SpMV kernel).
template <class T, class = void>
struct HasDistMark {
    static constexpr bool value = false;
};
template <class T>
struct HasDistMark<T, std::void_t<decltype(std::declval<const T&>().dist_mark(std::declval<const Params&>(),
                                                                                std::declval<Ctrl*>()))>> {
    static constexpr bool value = true;
};

// Optional per-Op shared-memory budget hint: `static constexpr int SMEM_CTAS`
// (resident CTAs per SM the stage ring is sized for).
template <class T, class = void>
struct SmemCtasOf {
    static constexpr int value = 0;
};
template <class T>
struct SmemCtasOf<T, std::void_t<decltype(T::SMEM_CTAS)>> {
    static constexpr int value = T::SMEM_CTAS;
};

// Optional Op member `static const double* early_vec(const Params&, int v)`:
// the staged vectors as a function of P alone — the steady-state vec() or a
// superset of it (extra streams are loaded and ignored). The producer then
// issues the first NS stages' vectors right after griddepcontrol.wait,
// overlapping the chained scalar prologue and enter() instead of following
// them (cgvk_stream.cuh k_stream).
#ifndef CGVK_EARLY
#define CGVK_EARLY 2         // stages whose vectors are issued right after the wait
#endif
template <class T, class = void>
struct HasEarlyVec {
    static constexpr bool value = false;
};
template <class T>
struct HasEarlyVec<T, std::void_t<decltype(T::early_vec(std::declval<const Params&>(), 0))>> {
    static constexpr bool value = true;
};

// `static constexpr bool NO_BAND = true`: an Op of the CSR engine only (no
// band-engine instantiation); `NO_PEER = true`: no peer-memory rank form.
template <class T, class = void>
struct NoBand {
    static constexpr bool value = false;
};
template <class T>
struct NoBand<T, std::void_t<decltype(T::NO_BAND)>> {
    static constexpr bool value = T::NO_BAND;
};
// One-kernel iterations (PrF, cgvk_variants.cuh). `early_vec(P, v, b)`: the
// staged vectors as a function of P and the buffer-set bit b = ctrl->pcur as
// this launch will see it — the producer works it out from the incoming
// control block itself (the predecessor toggles it iff it stepped), so the
// first stages' vectors are issued right after the wait, not after the
// chained prologue.
template <class T, class = void>
struct HasEarlyPcur {
    static constexpr bool value = false;
};
template <class T>
struct HasEarlyPcur<T, std::void_t<decltype(T::early_vec(std::declval<const Params&>(), 0, false))>> {
    static constexpr bool value = true;
};
#ifndef CGVK_K1_MIN_CTAS
#define CGVK_K1_MIN_CTAS 1  // register budget of the update kernels (resident CTAs)
#endif
// Optional `static constexpr int MINB`: resident CTAs per SM the register
// budget of the Op's kernel is sized for (__launch_bounds__).
template <class T, class = void>
struct MinbOf {
    static constexpr int value = T::CSR ? CGVK_SPMV_MIN_CTAS : CGVK_K1_MIN_CTAS;
};
template <class T>
struct MinbOf<T, std::void_t<decltype(T::MINB)>> {
    static constexpr int value = T::MINB;
};
template <class T, class = void>
struct NoPeer {
    static constexpr bool value = false;
};
template <class T>
struct NoPeer<T, std::void_t<decltype(T::NO_PEER)>> {
    static constexpr bool value = T::NO_PEER;
};
// Optional per-Op ring-depth hint: `static constexpr int STAGES`.
template <class T, class = void>
struct StagesOf {
    static constexpr int value = 0;
};
template <class T>
struct StagesOf<T, std::void_t<decltype(T::STAGES)>> {
    static constexpr int value = T::STAGES;
};

struct StageCfg {
    int nstage;     // ring depth
    int cap;        // CSR entries per stage (multiple of 4)
    int nvec;       // staged vectors
    int stage_bytes;
    int gvirt;      // Gv
    int ring;       // band engine: window ring tiles (2H + nstage)
    int pf;         // band engine: L2 prefetch distance (tiles)
    int chain;      // chained schedule: CH_* bits (0: last-CTA finish, in place)
    int gprev;      // chained schedule: the predecessor's Gv (its partials)
    unsigned int p2p_push;  // peer ranks: physical halo slots this launch pushes (kPushPnew: HS's p_new)
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// 1D bulk copy global -> shared, completion counted on `bar` (bytes % 16 == 0,
// both addresses 16-byte aligned). Streams are read once: evict-first in L2.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
    if (policy == 0) {  // default L2 policy
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(dst)),
            "l"(src), "r"(bytes), "r"(smem_u32(bar))
            : "memory");
        return;
    }
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ uint64_t evict_last_policy() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// L2 policy of a pipeline's matrix stream: 0/1 evict-first (streamed once per
// iteration), 2 none, 3 evict-last (an A that fits L2 with the vectors stays
// resident across iterations; chosen per matrix by size)
__device__ __forceinline__ uint64_t matrix_policy(int l2pol) {
    return l2pol < 2 ? evict_first_policy() : l2pol == 3 ? evict_last_policy() : 0;
}

__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory"); }

// Canonical CTA tree over the 256 consumer threads (same order as cta_tree).
// `mask` (uniform over the CTA): the dots in use — the others are skipped
// (their v[] is left as it is; nobody reads it).
template <int ND>
__device__ __forceinline__ void cta_tree_c(double (&v)[ND], double* sm, unsigned int mask = ~0u) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int d = 0; d < ND; ++d) {
        if (!((mask >> d) & 1u)) continue;
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) v[d] = ADD(v[d], __shfl_down_sync(0xffffffffu, v[d], off));
    }
    if (lane == 0) {
#pragma unroll
        for (int d = 0; d < ND; ++d)
            if ((mask >> d) & 1u) sm[d * 32 + warp] = v[d];
    }
    consumer_sync();
    if (warp == 0) {
#pragma unroll
        for (int d = 0; d < ND; ++d) {
            if (!((mask >> d) & 1u)) continue;
            double y = lane < kWarps ? sm[d * 32 + lane] : 0.0;
#pragma unroll
            for (int off = kWarps / 2; off >= 1; off >>= 1) y = ADD(y, __shfl_down_sync(0xffffffffu, y, off));
            v[d] = y;
        }
    }
    consumer_sync();
}

// Optional Op member `static unsigned int dmask(const Params&)`: the dot
// products this configuration uses, as a function of the solver's flags
// alone (CG-CG / GV: two of their five only with unsimplified_mu). A
// single-GPU chained kernel skips the others' trees and partial stores, its
// successor their loads and fold (measured per dot: 0.06 us per tree, 0.14 us
// in the successor's prologue; CG-CG P2D 7.3 -> 6.9 us, P64 12.7 -> 12.3, GV
// P64 15.0 -> 14.6). The PR family, which would skip one dot of six, measured
// slower with the predicates (P2D PR 7.5 -> 7.8, pipe-PR 7.8 -> 8.3 us) and
// declares no mask.
template <class T, class = void>
struct DmaskOf {
    __device__ static unsigned int get(const Params&) { return ~0u; }
};
template <class T>
struct DmaskOf<T, std::void_t<decltype(T::dmask(std::declval<const Params&>()))>> {
    __device__ static unsigned int get(const Params& P) { return T::dmask(P); }
};

__device__ __forceinline__ bool arrive_last_c(unsigned int* counter, int* flag) {
    consumer_sync();
    if (threadIdx.x == 0) {
        // (measured: a release add instead of fence + add changes nothing)
        __threadfence();
        const unsigned int prev = atomicAdd(counter, 1u);
        *flag = prev == gridDim.x - 1;
    }
    consumer_sync();
    const bool last = *flag != 0;
    if (last) __threadfence();
    return last;
}

// The row is consumed in chunks of 8 entries: all column and value loads of a
// chunk are issued first, then all of its gathers, then the in-order
// accumulation — so a row costs ~2 memory latencies, not 2 per entry. Loads
// past the row end are predicated off; nothing past it is ever multiplied.
#ifndef CGVK_CHUNK
#define CGVK_CHUNK 8
#endif
constexpr int kChunk = CGVK_CHUNK;

// A sparse row as seen by a thread: `len` entries, entry(k) = (column,
// value) of its k-th entry in CSR column order; a row is always summed left
// to right in that order (src/sparse_matrix.cpp:112-117).
// RowRef: CSR (stage or global), the row's entries contiguous.
struct RowRef {
    static constexpr int CH = kChunk;  // entries per chunk
    const double* va;
    const int* ci;
    int len;
    __device__ __forceinline__ void entry(int k, int& c, double& v) const {
        c = ci[k];
        v = va[k];
    }
};

#ifndef CGVK_BAND_LD
#define CGVK_BAND_LD 0  // slice loads: 0 ld.global.cs, 1 ld.global.nc, 2 ld.global.cg
#endif

// BandRow: the band engine's SELL-C-sigma slice (cgvk_band.cuh) — entry k of
// the thread's row at va[32 k], ci16[32 k] (the warp's 32 rows interleaved, so
// every load is one coalesced warp access), the column stored as a 16-bit
// offset from the tile's window base and returned as the index into the
// shared-memory window ring (tb + offset, wrapped once at RW).
template <int CHN>
struct BandRow {
    static constexpr int CH = CHN;
    const double* va;
    const unsigned short* ci;
    int len, tb, rw;
    __device__ __forceinline__ void entry(int k, int& c, double& v) const {
#if CGVK_BAND_LD == 1
        v = __ldg(va + 32 * k);
        int q = tb + static_cast<int>(__ldg(ci + 32 * k));
#elif CGVK_BAND_LD == 2
        v = __ldcg(va + 32 * k);
        int q = tb + static_cast<int>(__ldcg(ci + 32 * k));
#else
        v = __ldcs(va + 32 * k);
        int q = tb + static_cast<int>(__ldcs(ci + 32 * k));
#endif
        c = q >= rw ? q - rw : q;
    }
};


// Software-pipelined form (the band engine, whose matrix loads come from L2):
// the next chunk's column/value loads are issued before the current chunk is
// gathered and accumulated. The CSR engine reads its rows from the staged
// shared-memory tile and does not pipeline (measured neutral-to-slower).
template <class RR>
struct RowPipe {
    static constexpr bool value = false;
};
template <int C>
struct RowPipe<BandRow<C>> {
    static constexpr bool value = true;
};

template <class RR, class XF>
struct ChunkBuf {
    static constexpr int kC = RR::CH;
    int c[kC];
    double v[kC], x[kC];
    // column/value loads of entries k0 .. k0+7
    __device__ __forceinline__ void fetch(const RR& R, int k0) {
#pragma unroll
        for (int u = 0; u < RR::CH; ++u) {
            c[u] = -1;
            v[u] = 0.0;
            if (k0 + u < R.len) R.entry(k0 + u, c[u], v[u]);
        }
    }
    // the gathers (depend on the columns)
    __device__ __forceinline__ void resolve(XF xf) {
#pragma unroll
        for (int u = 0; u < RR::CH; ++u) x[u] = c[u] >= 0 ? xf(c[u]) : 0.0;
    }
    __device__ __forceinline__ void accumulate(double& sum) const {
#pragma unroll
        for (int u = 0; u < RR::CH; ++u)
            if (c[u] >= 0) sum = ADD(sum, MUL(v[u], x[u]));
    }
};

template <class RR, class XF>
__device__ __forceinline__ double row_dot(const RR& R, XF xf) {
    double sum = 0.0;
    if constexpr (RowPipe<RR>::value) {
        // chunk c+1's loads are in flight while chunk c is gathered and summed
        if (R.len <= 0) return sum;
        ChunkBuf<RR, XF> a, b;
        a.fetch(R, 0);
        for (int k0 = 0;; k0 += 2 * RR::CH) {
            const bool more_b = k0 + RR::CH < R.len;
            if (more_b) b.fetch(R, k0 + RR::CH);
            a.resolve(xf);
            a.accumulate(sum);
            if (!more_b) break;
            const bool more_a = k0 + 2 * RR::CH < R.len;
            if (more_a) a.fetch(R, k0 + 2 * RR::CH);
            b.resolve(xf);
            b.accumulate(sum);
            if (!more_a) break;
        }
    } else {
        for (int k0 = 0; k0 < R.len; k0 += RR::CH) {
            ChunkBuf<RR, XF> a;
            a.fetch(R, k0);
            a.resolve(xf);
            a.accumulate(sum);
        }
    }
    return sum;
}

// Two products over one traversal of the row (same per-product order).
// Pipelining it (CGVK_ROW2_PIPE=1) measured slower on R4M (register pressure).
#ifndef CGVK_ROW2_PIPE
#define CGVK_ROW2_PIPE 0
#endif
template <class RR, class XF1, class XF2>
struct ChunkBuf2 {
    static constexpr int kC = RR::CH;
    int c[kC];
    double v[kC], x1[kC], x2[kC];
    __device__ __forceinline__ void fetch(const RR& R, int k0) {
#pragma unroll
        for (int u = 0; u < kC; ++u) {
            c[u] = -1;
            v[u] = 0.0;
            if (k0 + u < R.len) R.entry(k0 + u, c[u], v[u]);
        }
    }
    __device__ __forceinline__ void resolve(XF1 f1, XF2 f2) {
#pragma unroll
        for (int u = 0; u < kC; ++u) {
            x1[u] = c[u] >= 0 ? f1(c[u]) : 0.0;
            x2[u] = c[u] >= 0 ? f2(c[u]) : 0.0;
        }
    }
    __device__ __forceinline__ void accumulate(double& s1, double& s2) const {
#pragma unroll
        for (int u = 0; u < kC; ++u)
            if (c[u] >= 0) {
                s1 = ADD(s1, MUL(v[u], x1[u]));
                s2 = ADD(s2, MUL(v[u], x2[u]));
            }
    }
};

template <class RR, class XF1, class XF2>
__device__ __forceinline__ void row_dot2(const RR& R, XF1 xf1, XF2 xf2, double& y1, double& y2) {
    double s1 = 0.0, s2 = 0.0;
    if constexpr (RowPipe<RR>::value && CGVK_ROW2_PIPE) {
        if (R.len > 0) {
            ChunkBuf2<RR, XF1, XF2> a, b;
            a.fetch(R, 0);
            for (int k0 = 0;; k0 += 2 * RR::CH) {
                const bool more_b = k0 + RR::CH < R.len;
                if (more_b) b.fetch(R, k0 + RR::CH);
                a.resolve(xf1, xf2);
                a.accumulate(s1, s2);
                if (!more_b) break;
                const bool more_a = k0 + 2 * RR::CH < R.len;
                if (more_a) a.fetch(R, k0 + 2 * RR::CH);
                b.resolve(xf1, xf2);
                b.accumulate(s1, s2);
                if (!more_a) break;
            }
        }
    } else {
        for (int k0 = 0; k0 < R.len; k0 += RR::CH) {
            ChunkBuf2<RR, XF1, XF2> a;
            a.fetch(R, k0);
            a.resolve(xf1, xf2);
            a.accumulate(s1, s2);
        }
    }
    y1 = s1;
    y2 = s2;
}

// Per-row input accessor handed to Op::row by the CSR pipeline: in(v) =
// staged vector v at the thread's own row; in.gather(k, j, g) = gathered
// operand k at column j, read from global g through L1/L2 (measured on B200,
// profiles/r01: for stencils L1 serves the +-1/+-N neighbours better than a
// shared-memory lookup with its divergent in-tile select).
struct StagedIn {
    const double* sv;  // stage vectors + own row
    __device__ __forceinline__ double operator()(int v) const { return sv[v * kBlock]; }
    __device__ __forceinline__ double gather(int, int j, const double* __restrict__ g) const {
        return __ldg(g + j);
    }
    // HS: p_j = r~_j + beta p_old_j formed at the gather
    __device__ __forceinline__ double gather_p(int j, const double* __restrict__ rt, const double* __restrict__ po,
                                               double beta) const {
        return ADD(__ldg(rt + j), MUL(beta, __ldg(po + j)));
    }
};

// Boundary tiles of peer-memory ranks (cgvk_p2p.cuh): the thread has just
// written its row's halo entries from the stamped receive buffers into the
// vector's halo region, so those tiles gather through L2 (ld.global.cg), not
// the non-coherent L1 path.
struct StagedInL2 {
    const double* sv;
    __device__ __forceinline__ double operator()(int v) const { return sv[v * kBlock]; }
    __device__ __forceinline__ double gather(int, int j, const double* __restrict__ g) const {
        return __ldcg(g + j);
    }
    __device__ __forceinline__ double gather_p(int j, const double* __restrict__ rt, const double* __restrict__ po,
                                               double beta) const {
        return ADD(__ldcg(rt + j), MUL(beta, __ldcg(po + j)));
    }
};

// Optional Op trait for the band engine: `static constexpr bool BAND_XF` — the
// window holds band_xf(source 0, source 1) instead of the NG raw sources.
template <class T, class = void>
struct BandXf {
    static constexpr bool value = false;
};
template <class T>
struct BandXf<T, std::void_t<decltype(T::BAND_XF)>> {
    static constexpr bool value = T::BAND_XF;
};

// Per-stage shared-memory layout: row_ptr slice, values, int32 columns,
// vectors.
struct StageView {
    int* rp;       // kRpInts
    double* va;    // cap
    int* ci;       // cap
    double* vec;   // nvec * kBlock
};

__device__ __forceinline__ StageView stage_view(unsigned char* base, const StageCfg& S, int slot) {
    unsigned char* p = base + (size_t)slot * S.stage_bytes;
    StageView v;
    v.rp = reinterpret_cast<int*>(p);
    p += kRpInts * 4;
    v.va = reinterpret_cast<double*>(p);
    p += (size_t)S.cap * 8;
    v.ci = reinterpret_cast<int*>(p);
    p += (size_t)S.cap * 4;
    v.vec = reinterpret_cast<double*>(p);
    return v;
}

__host__ __device__ inline int stage_bytes_for(int cap, int nvec, bool csr) {
    return kRpInts * 4 + (csr ? cap * 12 : 0) + nvec * kBlock * 8;
}

// Header in dynamic shared memory: barriers + per-slot metadata.
struct PipeHeader {
    uint64_t full[kMaxStages];
    uint64_t empty[kMaxStages];
    int k0a[kMaxStages];   // first staged value index (even)
    int k0c[kMaxStages];   // first staged column index (multiple of 4)
    int direct[kMaxStages];
    int last_flag;
    int pad[3];
    double red[kMaxDots * 32];
    uint64_t fold_bar;           // last CTA: bulk copy of the partials into the idle ring
    uint64_t pad2;
    uint64_t cfull[2], cempty[2];  // band engine: the per-row contribution buffers (cgvk_band.cuh)
    Ctrl cs;                     // last CTA: the control block finish() works on
};


// Last CTA: thread t sums partials q = t, t+256, ... in that order (the
// canonical fold); all loads are issued before the in-order adds so the fold
// costs one L2 latency, not Gv/256 of them.
constexpr int kFoldMax = 8;  // Gv <= 256 * 8
template <int ND>
__device__ __noinline__ void fold_partials(const double* part, int Gv, int t, double (&tot)[ND]) {
    for (int q0 = 0; q0 < Gv; q0 += kConsumers * kFoldMax) {
        double buf[kFoldMax][ND];
#pragma unroll
        for (int u = 0; u < kFoldMax; ++u) {
            const int q = q0 + t + u * kConsumers;
#pragma unroll
            for (int d = 0; d < ND; ++d) buf[u][d] = q < Gv ? __ldcg(part + d * Gv + q) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kFoldMax; ++u) {
            if (q0 + t + u * kConsumers < Gv) {
#pragma unroll
                for (int d = 0; d < ND; ++d) tot[d] = ADD(tot[d], buf[u][d]);
            }
        }
    }
}

// Last CTA, all consumer threads: the partials of every virtual CTA, folded in
// the canonical order (thread t: q = t, t+256, ...). When they fit the idle
// stage ring they arrive with ONE bulk copy (one L2 latency, no registers);
// otherwise fold_partials issues the loads from registers.
template <int ND>
__device__ __forceinline__ void fold_last(const double* part, int Gv, int t, PipeHeader* H, unsigned char* ring,
                                          size_t ring_bytes, double (&tot)[ND]) {
    // dots [0, nb) by one bulk copy; up to two more from registers, their loads
    // issued before the bulk wait so both take one L2 latency together
    constexpr int kRegDots = 2;
    if (Gv <= kConsumers) {
        // small grids (rank shards): one partial per thread and dot, all loads
        // in flight together — one L2 round trip, no proxy fence, no barrier
        double v[ND];
#pragma unroll
        for (int d = 0; d < ND; ++d) v[d] = t < Gv ? __ldcg(part + (size_t)d * Gv + t) : 0.0;
        if (t < Gv) {
#pragma unroll
            for (int d = 0; d < ND; ++d) tot[d] = ADD(tot[d], v[d]);
        }
        return;
    }
    const size_t per_dot = (size_t)Gv * 8;
    const int nb = (int)min((size_t)ND, ring_bytes / per_dot);
    if (ND - nb > kRegDots || Gv > kConsumers * kFoldMax) {
        fold_partials<ND>(part, Gv, t, tot);
        return;
    }
    if (t == 0 && nb > 0) {
        // the partials were written by other CTAs (generic proxy, released by
        // their fences + the arrival atomic); order them before the bulk read
        const uint32_t bytes = (uint32_t)((nb * per_dot + 15) & ~(size_t)15);
        asm volatile("fence.proxy.async.global;" ::: "memory");
        mbar_expect_tx(&H->fold_bar, bytes);
        bulk_g2s(ring, part, bytes, &H->fold_bar, 0);
    }
    double rv[kRegDots][kFoldMax];
#pragma unroll
    for (int e = 0; e < kRegDots; ++e) {
        const int d = nb + e;
#pragma unroll
        for (int u = 0; u < kFoldMax; ++u) {
            const int q = t + u * kConsumers;
            rv[e][u] = (d < ND && q < Gv) ? __ldcg(part + (size_t)d * Gv + q) : 0.0;
        }
    }
    if (nb > 0) mbar_wait(&H->fold_bar, 0);
    const double* sp = reinterpret_cast<const double*>(ring);
#pragma unroll
    for (int u = 0; u < kFoldMax; ++u) {
        const int q = t + u * kConsumers;
        if (q >= Gv) break;
#pragma unroll
        for (int d = 0; d < ND; ++d) {
            const double v = d < nb ? sp[d * Gv + q] : rv[(d - nb) < kRegDots ? d - nb : 0][u];
            tot[d] = ADD(tot[d], v);
        }
    }
}

// Last CTA, all consumer threads: op.finish on a shared-memory copy of the
// control block (its read-modify-writes then cost shared-memory latency, not
// a chain of L2 round trips); only the 4-byte words finish changed are
// written back, so a concurrent finalize of a row-partitioned solve (GV /
// pipe-PR: k_finalize on the side stream while K2 ends) never sees its
// fields overwritten with a stale copy, and the arrival counters stay as the
// atomics left them.
constexpr int kCtrlWords = sizeof(Ctrl) / 16;
template <class Op>
__device__ __forceinline__ void finish_last(const Op& op, const Params& P, PipeHeader* H, const double* tot, int t) {
    uint4* cs = reinterpret_cast<uint4*>(&H->cs);
    uint4* cg = reinterpret_cast<uint4*>(P.ctrl);
    uint4 orig = make_uint4(0, 0, 0, 0);
    if (t < kCtrlWords) {
        orig = __ldcg(cg + t);
        cs[t] = orig;
    }
    consumer_sync();
    if (t == 0) op.finish(P, &H->cs, tot);
    consumer_sync();
    if (t < kCtrlWords) {
        const uint4 now = cs[t];
        unsigned int* dst = reinterpret_cast<unsigned int*>(cg + t);
        if (now.x != orig.x) dst[0] = now.x;
        if (now.y != orig.y) dst[1] = now.y;
        if (now.z != orig.z) dst[2] = now.z;
        if (now.w != orig.w) dst[3] = now.w;
    }
}

// ------------------------------------------------------ chained schedule
//
// The last-CTA schedule ends every reducing kernel with a chain of round
// trips on its critical path: a fence and the arrival atomic, the fold of
// all partials, a load of the control block, the scalar tail, the
// write-back, the kernel's end — and only then may the next kernel read a
// scalar. In the chained schedule a reducing kernel's CTAs stop at their
// partials; every CTA of the NEXT kernel, right after griddepcontrol.wait,
// loads the control block and the partials together, folds them in the
// canonical order and runs the predecessor's finish — the same scalar code
// on the same bits in every CTA (measured: P64 61.1 k -> 66.9 k it/s, P2D
// 86.7 k -> 96.4 k against the last CTA folding into the control block). A
// kernel whose finish needs no dots (sync() == 1) does not arrive at all.
// Control block and partials are double-buffered: K1 reads `ctrl` / `part`
// and writes `ctrl_b` (CTA 0) / `part_b`; K2 the other way round (no kernel
// reads the copy it writes). A graph of chained iterations ends with
// k_chain_tail (one CTA), which finishes the last K2 and leaves `ctrl`
// complete, as the last-CTA schedule does. Peer-memory ranks keep a last CTA
// per rank: it publishes the rank total (cgvk_p2p.cuh).
#ifndef CGVK_TIMELINE
#define CGVK_TIMELINE 0
#endif
#if CGVK_TIMELINE
__device__ unsigned long long g_timeline[2][1024][8];
#endif
__device__ __forceinline__ void tl_mark(int kernel, int slot) {
#if CGVK_TIMELINE
    if (threadIdx.x == 0 && blockIdx.x < 1024) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_timeline[kernel][blockIdx.x][slot] = t;
    }
#endif
}

constexpr int CH_ON = 1;    // chained: totals only, the successor finishes
constexpr int CH_FOLD = 2;  // run the predecessor's finish first
constexpr int CH_ODD = 4;   // the iteration's second kernel (K2)

__device__ __forceinline__ Params with_ctrl(const Params& P, Ctrl* c) {
    Params Q = P;
    Q.ctrl = c;
    return Q;
}

constexpr int kSuccFoldMax = 2 * kConsumers;  // predecessor partials per register pass
// Every CTA of the successor reads the same partials (ND x Gv doubles: hot
// lines in L2). CGVK_FOLD_L1=1 reads them through L1, so the CTAs resident on
// one SM share one L2 read (the non-coherent path is safe here as it is for
// the SpMV gathers: the buffers were written by the previous kernel).
// Measured: P64 68.7 k -> 69.9 k it/s (pipe-PR 17.1 -> 16.4 us), P128 +0.3 %.
#ifndef CGVK_P2P_PLAN_PF
#define CGVK_P2P_PLAN_PF 1  // peer ranks: prefetch the exchange plan into L1 before the dependency wait
#endif
#ifndef CGVK_FOLD_L1
#define CGVK_FOLD_L1 1
#endif
#if CGVK_FOLD_L1
#define CGVK_FOLD_LD __ldg
#else
#define CGVK_FOLD_LD __ldcg
#endif
// The control block itself (256 bytes every CTA reads): CGVK_CTRL_L1=1 the same way.
#ifndef CGVK_CTRL_L1
#define CGVK_CTRL_L1 0
#endif
#if CGVK_CTRL_L1
#define CGVK_CTRL_LD __ldg
#else
#define CGVK_CTRL_LD __ldcg
#endif

// Words of the control block CTA 0 copies forward (the totals are written by
// the kernel's last CTA).
constexpr int kCtrlHead = offsetof(Ctrl, tot) / 16;

// All threads of the CTA. Warp 0 loads the control block into H->cs — one
// coalesced 256-byte load, not a bulk copy, which would queue behind the
// producer's matrix prefetch in the TMA unit; thread 0 runs the
// predecessor's finish on it; CTA 0 writes the advanced state to `out`.
//
// Single GPU: the predecessor's CTAs only wrote their
// partials (no arrival counter, no fence, no last CTA — griddepcontrol.wait
// already orders them before this kernel); the consumer warps of EVERY CTA
// fold them here in the canonical order (fold_partials + cta_tree_c: the
// same bits the last CTA produced), their loads issued together with the
// control-block load. `gprev` = the predecessor's virtual CTAs. The partial
// buffers are double-buffered like the control block (K1 writes `part_b`,
// K2 `part`), so a slow CTA still folding never sees its successor's writes.
//
// Peer-memory ranks (PEER, cgvk_p2p.cuh): the predecessor's totals are the
// rank-ordered sum of every rank's published total (waited for by stamp); a
// K2 whose predecessor has a dist_mark (GV / pipe-PR) takes the go-ahead and
// leaves the K1 reduction to the next K1 (`defer`), which folds it first with
// its own type (Self); `incr` advances the kernel sequence number.
template <class Self, class Prev, bool PEER = false>
__device__ __forceinline__ void chain_prologue(const Params& P, int chain, PipeHeader* H, Ctrl* out, int gprev,
                                               bool incr = true) {
    const int t = threadIdx.x;
    if constexpr (!PEER) {
        if (t < kConsumers) {
            constexpr int ND = Prev::ND > 0 ? Prev::ND : 1;
            constexpr int U = kSuccFoldMax / kConsumers;
            const bool fold = Prev::ND > 0 && (chain & CH_FOLD);
            const double* pin = (chain & CH_ODD) ? P.part_b : P.part;
            const unsigned int dm = DmaskOf<Prev>::get(P);  // the predecessor's dots in use
            double v[U][ND];
            auto load = [&](int q0) {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int q = q0 + t + u * kConsumers;
#pragma unroll
                    for (int d = 0; d < ND; ++d)
                        v[u][d] = (q < gprev && ((dm >> d) & 1u)) ? CGVK_FOLD_LD(pin + d * gprev + q) : 0.0;
                }
            };
            if (fold) load(0);  // issued before the control block arrives
            if (t < 32) {
                constexpr int kWords = sizeof(Ctrl) / 16;
                const uint4* in = reinterpret_cast<const uint4*>((chain & CH_ODD) ? P.ctrl_b : P.ctrl);
                if (t < kWords) reinterpret_cast<uint4*>(&H->cs)[t] = CGVK_CTRL_LD(in + t);
            }
            consumer_sync();
            tl_mark(Self::CSR, 7);
            if (chain & CH_FOLD) {
                Params Q = with_ctrl(P, &H->cs);
                if (blockIdx.x != 0) Q.hist = nullptr;  // side effects once
                Prev prev;
                const bool go = prev.enter(Q);  // read-only on the shared copy: uniform
                const int m = go ? prev.sync() : 0;
                double tot[ND];
#pragma unroll
                for (int d = 0; d < ND; ++d) tot[d] = 0.0;
                if (Prev::ND > 0 && m == 2) {
                    // thread t: q = t, t + 256, ... in order (fold_partials' order)
                    for (int q0 = 0; q0 < gprev; q0 += kSuccFoldMax) {
                        if (q0 > 0) load(q0);
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            if (q0 + t + u * kConsumers < gprev) {
#pragma unroll
                                for (int d = 0; d < ND; ++d) tot[d] = ADD(tot[d], v[u][d]);
                            }
                        }
                    }
                    cta_tree_c<ND>(tot, H->red, dm);
                }
                tl_mark(Self::CSR, 4);
                if (t == 0 && go && m != 0) prev.finish(Q, &H->cs, tot);
            }
        }
    } else if (t < 32) {
        constexpr int kWords = sizeof(Ctrl) / 16;
        if (t < kWords) reinterpret_cast<uint4*>(&H->cs)[t] = __ldcg(reinterpret_cast<const uint4*>((chain & CH_ODD) ? P.ctrl_b : P.ctrl) + t);
        __syncwarp();
        // warp 0: every lane evaluates the (read-only) enter() decisions on
        // the shared copy, the warp polls the exchanged totals together,
        // lane 0 runs finish(); __syncwarp between lane 0's writes and the
        // next reads
        unsigned int* scratch = reinterpret_cast<unsigned int*>(H->red);
        if (chain & CH_FOLD) {
            Params Q = with_ctrl(P, &H->cs);
            if (blockIdx.x != 0) Q.hist = nullptr;
            if constexpr (HasDistMark<Self>::value) {
                if (H->cs.defer) {  // the K1 reduction one iteration back (GV / pipe-PR)
                    Self self;
                    const bool go = self.enter(Q) && self.sync() == 2;
                    double tot[kMaxDots];
                    if (go) p2p_fold_totals<Self::ND>(P.pp, H->cs.dstamp, tot, scratch);
                    if (t == 0) {
                        if (go) self.finish(Q, &H->cs, tot);
                        H->cs.defer = 0;
                    }
                    __syncwarp();
                }
            }
            Prev prev;
            if (prev.enter(Q)) {
                const int m = prev.sync();
                if (m == 2) {
                    bool deferred = false;
                    if constexpr (HasDistMark<Prev>::value) {
                        if (chain & CH_ODD) {  // K2: take the go-ahead, the next K1 folds
                            if (t == 0) {
                                prev.dist_mark(Q, &H->cs);
                                H->cs.defer = 1;
                                H->cs.dstamp = H->cs.hseq;
                            }
                            deferred = true;
                        }
                    }
                    if (!deferred) {
                        double tot[kMaxDots];
                        p2p_fold_totals<Prev::ND>(P.pp, H->cs.hseq, tot, scratch);
                        if (t == 0) prev.finish(Q, &H->cs, tot);
                    }
                } else if (m == 1) {
                    const double none[kMaxDots] = {};
                    if (t == 0) prev.finish(Q, &H->cs, none);
                }
            }
            __syncwarp();
        }
        if (t == 0 && incr) H->cs.hseq += 1;
    }
    __syncthreads();
    if (blockIdx.x == 0 && t < kCtrlHead)
        reinterpret_cast<uint4*>(out)[t] = reinterpret_cast<const uint4*>(&H->cs)[t];
}

// The chained graph's last node: the final K2's scalar tail (and, on
// peer-memory ranks, a GV / pipe-PR K1 reduction K2 deferred).
// Launched with kConsumers threads (the successor fold's canonical tree).
template <class Op1, class Op2, bool PEER = false>
__global__ void __launch_bounds__(kConsumers) k_chain_tail(Params P, StageCfg S) {
    __shared__ __align__(128) PipeHeader H;
    asm volatile("griddepcontrol.wait;" ::: "memory");
    // (S.chain & CH_ODD: the last kernel was an even one — a one-kernel
    // iteration schedule after an odd number of launches — and wrote ctrl_b)
    chain_prologue<Op1, Op2, PEER>(P, CH_ON | CH_FOLD | (S.chain & CH_ODD), &H, P.ctrl, S.gprev, /*incr=*/false);
}

// Programmatic dependent launch: wait for the preceding kernel's results /
// allow the next kernel to start its prologue. CGVK_PDL_LATE=1 signals the
// dependents only when a CTA has finished its tiles (before the reduction
// tail) instead of right after the wait.
// Measured (profiles/r01): late helps HS (two short kernels, both with a
// reduction: P128 72.6 -> 71.0 us, P64 24.1 -> 21.7 us), early helps the
// others; an Op opts in with `static constexpr bool PDL_LATE = true`.
#ifndef CGVK_PDL_LATE
#define CGVK_PDL_LATE 0
#endif
template <class T, class = void>
struct PdlLate {
    static constexpr bool value = CGVK_PDL_LATE != 0;
};
template <class T>
struct PdlLate<T, std::void_t<decltype(T::PDL_LATE)>> {
    static constexpr bool value = T::PDL_LATE;
};
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Add expected bytes without arriving (the stage's single arrival comes later).
__device__ __forceinline__ void mbar_expect_tx_only(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

// Issue the CSR part of `tile` into `slot`: row_ptr slice, values, columns
// (or mark the tile "direct" when it exceeds the stage capacity).
__device__ __forceinline__ void stage_csr(const Params& P, const StageCfg& S, PipeHeader* H,
                                          unsigned char* stages, int slot, int tile, uint64_t pol,
                                          bool) {
    StageView V = stage_view(stages, S, slot);
    const int r0 = tile * kBlock;
    const int rows = min(kBlock, P.n - r0);
    const uint32_t rp_bytes = ((rows + 1) * 4 + 15) & ~15;
    const int k0 = __ldg(P.rp + r0), k1 = __ldg(P.rp + r0 + rows);
    const int k0a = k0 & ~1, k0c = k0 & ~3;  // 16-byte aligned bulk sources
    const bool direct = k1 - k0c + 4 > S.cap;
    const uint32_t va_bytes = direct ? 0u : (((k1 - k0a) * 8 + 15) & ~15);
    const uint32_t ci_bytes = direct ? 0u : (((k1 - k0c) * 4 + 15) & ~15);
    H->k0a[slot] = k0a;
    H->k0c[slot] = k0c;
    H->direct[slot] = direct;
    mbar_expect_tx_only(&H->full[slot], rp_bytes + va_bytes + ci_bytes);
    bulk_g2s(V.rp, P.rp + r0, rp_bytes, &H->full[slot], pol);
    if (!direct) {
        bulk_g2s(V.va, P.va + k0a, va_bytes, &H->full[slot], pol);
        bulk_g2s(V.ci, P.ci + k0c, ci_bytes, &H->full[slot], pol);
    }
}

// ---------------------------------------------------------------- driver
//
// Op contract (all device members):
//   static constexpr int NV, ND; static constexpr bool CSR;
//   bool enter(const Params&)            uniform: false -> nothing to do
//   const double* vec(const Params&, int v)   stream v (nullptr: not staged)
//   int sync()                           0: none, 1: arrive only, 2: reduce ND dots
//   void row(const Params&, int i, const In& in, const RowRef&, double* acc)
//        in(v) = staged value of vector v at row i, in.gather(v, j, g) = column j
//   void finish(const Params&, Ctrl*, const double* tot)   thread 0, last CTA
// MINB: resident CTAs the register budget is sized for. The SpMV kernels use
// CGVK_SPMV_MIN_CTAS when their stage lets that many CTAs fit, else 1 — a
// long-row matrix (R4M, ~27 entries/row) whose 2-stage ring already fills the
// SM gets the registers to keep a whole chunk of gathers in flight.
// CGVK_TIMELINE=1 (A/B builds only): per-CTA %globaltimer stamps of the
// kernel's phases, read back with cgvk_debug_timeline.
// Prev: the other kernel of the iteration (chained schedule: its partials
// are folded here, see chain_prologue).
// Two virtual CTAs per physical CTA (order 0; the register-bound update
// kernels of GV / pipe-PR run 2 CTAs/SM against G = 3 x SMs): their tiles are
// interleaved — step s takes vCTA s & 1's tile s >> 1 — so the grid still
// sweeps the tiles in one monotonic pass (tile p + Gp s). Each virtual CTA
// keeps its own accumulators, so its tiles are still summed in order: the
// bits are those of the sequential schedule. Returns the tile, -1 (vCTA 1
// has no tile at this step) or -2 (done).
// Opt-in per Op (`static constexpr bool RR2 = true`): measured P128 pipe-PR
// 87.1 -> 84.6 us, V256 657 -> 646 us; GV's K1 loses 1.3 us (off there).
#ifndef CGVK_RR2
#define CGVK_RR2 1
#endif
template <class T, class = void>
struct Rr2Of {
    static constexpr bool value = false;
};
template <class T>
struct Rr2Of<T, std::void_t<decltype(T::RR2)>> {
    static constexpr bool value = T::RR2 && CGVK_RR2 != 0;
};
__device__ __forceinline__ int rr2_tile(int p, int Gp, int Gv, int ntiles, int s) {
    const int jt = s >> 1;
    if (p + jt * Gv >= ntiles) return -2;
    const int tile = p + (s & 1) * Gp + jt * Gv;
    return tile < ntiles ? tile : -1;
}

// Reversed sweep (Op trait `REVERSE = true`, kernels without dot products,
// so the tile order changes no bit): the CTA walks its tiles p + Gp s from
// the highest s down. The other kernel of the iteration sweeps upwards, so
// each kernel starts on the tiles its predecessor wrote last — still in L2.
#ifndef CGVK_REVERSE
#define CGVK_REVERSE 1
#endif
template <class T, class = void>
struct RevOf {
    static constexpr bool value = false;
};
template <class T>
struct RevOf<T, std::void_t<decltype(T::REVERSE)>> {
    static_assert(!T::REVERSE || T::ND == 0, "a reversed sweep would reorder the dot products");
    static constexpr bool value = T::REVERSE && CGVK_REVERSE != 0;
};

// L2 policy of a staged vector: streams are read once (evict-first), but an
// SpMV kernel's staged copy of its gathered operand is gathered again by the
// tiles +-N^2 rows away — kept at normal priority (measured V256 +2.6 %,
// HS 495 -> 471 us; CGVK_GATHER_NORMAL=0 restores evict-first).
#ifndef CGVK_GATHER_NORMAL
#define CGVK_GATHER_NORMAL 1
#endif
template <class Op>
__device__ __forceinline__ uint64_t staged_policy(const Op& op, const Params& P, const double* src, uint64_t vpol) {
    if constexpr (Op::CSR && CGVK_GATHER_NORMAL) {
#pragma unroll
        for (int k = 0; k < Op::NG; ++k)
            if (src == op.gsrc(P, k)) return 0;
    }
    return vpol;
}

template <class Op, class Prev, bool PEER>
__device__ __forceinline__ void stream_body(const Params& P, const StageCfg& S);

// PEER: the peer-memory rank form (cgvk_p2p.cuh), a separate instantiation so
// the single-GPU kernels carry none of its code or registers.
template <class Op, class Prev, int MINB = MinbOf<Op>::value, bool PEER = false>
__global__ void __launch_bounds__(kThreads, MINB) k_stream(Params P, StageCfg S) {
    stream_body<Op, Prev, PEER>(P, S);
}

// The same kernel under an explicit register cap (__maxnreg__ cannot be
// combined with __launch_bounds__): for an Op with `static constexpr int
// MAXNREG` (cgvk_api.cu make_launch picks it).
template <class T, class = void>
struct MaxnregOf {
    static constexpr int value = 0;
};
template <class T>
struct MaxnregOf<T, std::void_t<decltype(T::MAXNREG)>> {
    static constexpr int value = T::MAXNREG;
};
template <class Op, class Prev, bool PEER = false>
__global__ void __maxnreg__(MaxnregOf<Op>::value > 0 ? MaxnregOf<Op>::value : 255) k_stream_nr(Params P, StageCfg S) {
    stream_body<Op, Prev, PEER>(P, S);
}

template <class Op, class Prev, bool PEER>
__device__ __forceinline__ void stream_body(const Params& P, const StageCfg& S) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    PipeHeader* H = reinterpret_cast<PipeHeader*>(smem_raw);
    unsigned char* stages = smem_raw + ((sizeof(PipeHeader) + 127) / 128) * 128;
    const int Gv = S.gvirt, Gp = gridDim.x, ntiles = P.ntiles, NS = S.nstage;
    const int warp = threadIdx.x >> 5;
    const bool producer = threadIdx.x == kConsumers;  // lane 0 of the producer warp
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(&H->full[s], 1);
            mbar_init(&H->empty[s], kWarps);
        }
        mbar_init(&H->fold_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    // The matrix does not depend on the previous kernel: under programmatic
    // dependent launch the producer streams A for its first NS tiles while
    // that kernel is still finishing, then waits for it.
    uint64_t pol = 0;
    int npre = 0;
    // reversed sweep: the CTA's tiles are exactly p + Gp s when Gp divides Gv
    // (or every virtual CTA is one tile)
    const bool rev = RevOf<Op>::value && P.order == 0 && (Gv % Gp == 0 || Gv == ntiles);
    const int nrev = rev ? ((int)blockIdx.x < ntiles ? (ntiles - 1 - (int)blockIdx.x) / Gp + 1 : 0) : 0;
    const bool rr2 = Rr2Of<Op>::value && !Op::CSR && P.order == 0 && (int)blockIdx.x + Gp < Gv &&
                     (int)blockIdx.x + 2 * Gp >= Gv;
    constexpr bool kEarlyP = HasEarlyPcur<Op>::value && CGVK_EARLY > 0;
    constexpr bool kEarly = (HasEarlyVec<Op>::value || kEarlyP) && CGVK_EARLY > 0;
    int early_tile[kMaxStages];
    int nearly = 0;  // stages whose vectors are issued right after the wait
    if (producer && (Op::CSR || kEarly)) {
        if (Op::CSR) pol = matrix_policy(P.l2pol);
        int q = 0;
        if (rev) {
            for (int st = 0; st < nrev && q < NS; ++st) {
                const int tile = (int)blockIdx.x + Gp * (nrev - 1 - st);
                if (Op::CSR) stage_csr(P, S, H, stages, q, tile, pol, /*arrive=*/false);
                early_tile[q++] = tile;
            }
        } else if (rr2) {
            for (int st = 0; q < NS; ++st) {
                const int tile = rr2_tile(blockIdx.x, Gp, Gv, ntiles, st);
                if (tile == -2) break;
                if (tile >= 0) early_tile[q++] = tile;
            }
        } else {
            CGVK_FOR_VB(vb, P.order, blockIdx.x, Gv, Gp) {
                CGVK_FOR_TILE(tile, P.order, vb, ntiles, Gv) {
                    if (q == NS) break;
                    if (Op::CSR) stage_csr(P, S, H, stages, q, tile, pol, /*arrive=*/false);
                    early_tile[q++] = tile;
                }
                if (q == NS) break;
            }
        }
        if (Op::CSR) npre = q;
        if (kEarly) nearly = min(q, CGVK_EARLY);
    }
    if constexpr (PEER && CGVK_P2P_PLAN_PF) {
        // the exchange plan is immutable: its three lines into L1 while the
        // previous kernel drains, so the prologue's fold, the boundary rows
        // and the last CTA's publication read it at L1 latency
        if (threadIdx.x < (sizeof(PeerPlan) + 127) / 128)
            asm volatile("prefetch.global.L1 [%0];" ::"l"(reinterpret_cast<const char*>(P.pp) + 128 * threadIdx.x));
    }
    tl_mark(Op::CSR, 0);
    pdl_wait();
    tl_mark(Op::CSR, 1);
    if constexpr (kEarly) {
        if (producer) {
            const uint64_t vpol = P.l2pol == 0 ? (Op::CSR ? pol : evict_first_policy()) : 0;
            bool pb = false;  // kEarlyP: ctrl->pcur as this launch's enter() will see it
            if constexpr (kEarlyP) {
                const Ctrl* cin = (S.chain & CH_ODD) ? P.ctrl_b : P.ctrl;
                pb = __ldcg(&cin->pcur) != 0;
                if ((S.chain & CH_FOLD) && Prev::entered(cin))
                    pb = !pb;  // the predecessor ran: its finish (in the prologue) flips the set
            }
            auto evec = [&](int v) -> const double* {
                if constexpr (kEarlyP) return Op::early_vec(P, v, pb);
                else return Op::early_vec(P, v);
            };
            for (int q = 0; q < nearly; ++q) {
                StageView V = stage_view(stages, S, q);
                const int r0 = early_tile[q] * kBlock;
                const uint32_t vec_bytes = (min(kBlock, P.n - r0) * 8 + 15) & ~15;
                uint32_t bytes = 0;
#pragma unroll
                for (int v = 0; v < Op::NV; ++v)
                    if (evec(v)) bytes += vec_bytes;
                mbar_expect_tx(&H->full[q], bytes);  // + the stage's arrival
#pragma unroll
                for (int v = 0; v < Op::NV; ++v) {
                    const double* src = evec(v);
                    uint64_t vp = vpol;
                    if constexpr (!kEarlyP) vp = staged_policy(Op{}, P, src, vpol);
                    if (src) bulk_g2s(V.vec + v * kBlock, src + r0, vec_bytes, &H->full[q], vp);
                }
            }
        }
    }
    if (!PdlLate<Op>::value) pdl_trigger();
    const int chain = S.chain;
    if (chain) {
        chain_prologue<Op, Prev, PEER>(P, chain, H, (chain & CH_ODD) ? P.ctrl : P.ctrl_b, S.gprev);
        tl_mark(Op::CSR, 5);
    }
    Op op;
    if (!(chain ? op.enter(with_ctrl(P, &H->cs)) : op.enter(P))) {  // uniform over the grid
        if (PEER && threadIdx.x < kConsumers) {
            // peer ranks: the neighbours still get this kernel's stamp on the
            // (unchanged) boundary rows, as a single-GPU solve would read them
            // (HS: both p buffers — the next p_old is this kernel's p_old)
            const unsigned int mask = p2p_idle_mask(S.p2p_push, H->cs.pcur);
            const int tlo = P.pp->tlo, hif = P.pp->hi_first;
            CGVK_FOR_VB(vb, P.order, blockIdx.x, Gv, Gp) {
                CGVK_FOR_TILE(tile, P.order, vb, ntiles, Gv) {
                    if (mask && (tile < tlo || tile >= hif))
                        p2p_push_row(P.pp, mask, tile * kBlock + (int)threadIdx.x, P.n, H->cs.hseq);
                }
            }
        }
        if (producer) {  // drain the prefetch before the CTA exits
            for (int q = 0; q < max(npre, nearly); ++q) {
                if (q >= nearly) mbar_arrive(&H->full[q]);
                mbar_wait(&H->full[q], 0);
            }
        }
        return;
    }

    if (warp == kWarps) {  // ------------------------------ producer warp
        if (!producer) return;
        if (!Op::CSR) pol = P.l2pol < 2 ? evict_first_policy() : 0;  // vectors: never evict-last
        const double* vp[kMaxVec];
#pragma unroll
        for (int v = 0; v < Op::NV; ++v) vp[v] = op.vec(P, v);
        int j = 0;
        const uint64_t vpol = P.l2pol == 0 ? pol : 0;
        unsigned int normal_mask = 0;  // staged vectors kept at normal L2 priority
#pragma unroll
        for (int v = 0; v < Op::NV; ++v)
            if (vp[v] && staged_policy(op, P, vp[v], vpol) != vpol) normal_mask |= 1u << v;
        auto produce_tile = [&](int tile) {
            {
                if (j < nearly) {  // issued right after the wait
                    ++j;
                    return;
                }
                const int slot = j % NS;
                if (j >= NS) mbar_wait(&H->empty[slot], ((j / NS) - 1) & 1);
                StageView V = stage_view(stages, S, slot);
                const int r0 = tile * kBlock;
                const int rows = min(kBlock, P.n - r0);
                if (Op::CSR && j >= npre) stage_csr(P, S, H, stages, slot, tile, pol, false);
                const uint32_t vec_bytes = (rows * 8 + 15) & ~15;
                uint32_t bytes = 0;
#pragma unroll
                for (int v = 0; v < Op::NV; ++v)
                    if (vp[v]) bytes += vec_bytes;
                mbar_expect_tx(&H->full[slot], bytes);  // + this thread's arrival
#pragma unroll
                for (int v = 0; v < Op::NV; ++v)
                    if (vp[v])
                        bulk_g2s(V.vec + v * kBlock, vp[v] + r0, vec_bytes, &H->full[slot],
                                 (normal_mask >> v) & 1u ? 0ull : vpol);
                ++j;
            }
        };
        if (rev) {
            for (int st = 0; st < nrev; ++st) produce_tile((int)blockIdx.x + Gp * (nrev - 1 - st));
        } else if (rr2) {
            for (int st = 0;; ++st) {
                const int tile = rr2_tile(blockIdx.x, Gp, Gv, ntiles, st);
                if (tile == -2) break;
                if (tile >= 0) produce_tile(tile);
            }
        } else {
            CGVK_FOR_VB(vb, P.order, blockIdx.x, Gv, Gp) {
                CGVK_FOR_TILE(tile, P.order, vb, ntiles, Gv) produce_tile(tile);
            }
        }
        return;
    }

    // ------------------------------------------------------ consumer warps
    const int t = threadIdx.x;
    double acc[Op::ND > 0 ? Op::ND : 1];
    int j = 0;
    // peer ranks (cgvk_p2p.cuh): after a boundary tile, its rows of the pushed
    // vectors go to the neighbours (out of line: the common path only compares
    // the tile); before a boundary row, its halo entries come from the
    // receive buffers into the vector's halo region (p2p_unpack_row)
    const PeerPlan* const pp = P.pp;
    const int p2p_tlo = PEER ? __ldg(&pp->tlo) : 0, p2p_hif = PEER ? __ldg(&pp->hi_first) : 0x7fffffff;
    const int p2p_hb = PEER ? __ldg(&pp->hbase) : 0x7fffffff;
    const unsigned int p2p_h = PEER ? H->cs.hseq : 0u;
    const int p2p_pc = PEER ? H->cs.pcur : 0;
    const unsigned int p2p_mask = PEER ? p2p_push_mask(S.p2p_push, p2p_pc) : 0u;
    auto consume_tile = [&](int slot, int tile) {
        const bool pb = PEER && (tile < p2p_tlo || tile >= p2p_hif);
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
            if constexpr (PEER && Op::CSR) {
                if (pb) {  // this row's halo entries, then gathers through L2
                    if constexpr (HasEarlyPcur<Op>::value) {  // one-kernel iteration: three exchanged sources
                        p2p_unpack_row3(pp, R.ci, R.len, p2p_hb, p2p_pc, op.gsrc(P, 0), op.gsrc(P, 1), op.gsrc(P, 2),
                                        p2p_h);
                    } else {
                        const double* g0 = op.gsrc(P, 0);
                        const double* g1 = Op::NG > 1 ? op.gsrc(P, Op::NG - 1) : nullptr;
                        p2p_unpack_row(pp, R.ci, R.len, p2p_hb, g0, g1, p2p_h, p2p_pc);
                    }
                    op.row(P, i, StagedInL2{V.vec + t}, R, acc);
                } else {
                    op.row(P, i, StagedIn{V.vec + t}, R, acc);
                }
            } else {
                op.row(P, i, StagedIn{V.vec + t}, R, acc);
            }
        }
        __syncwarp();
        if ((t & 31) == 0) mbar_arrive(&H->empty[slot]);
        if (pb && p2p_mask) p2p_push_row(pp, p2p_mask, i, P.n, p2p_h);
    };
    double* const part = (!PEER && chain && !(chain & CH_ODD)) ? P.part_b : P.part;
    // (single-GPU chained kernels: only the dots in use — the successor folds
    // exactly those; every other schedule folds all ND partial arrays)
    const unsigned int dm = (!PEER && chain) ? DmaskOf<Op>::get(P) : ~0u;
    auto close_vb = [&](int vb) {
        if constexpr (Op::ND > 0) {
            if (op.sync() != 2) return;
            cta_tree_c<Op::ND>(acc, H->red, dm);
            if (t == 0) {
#pragma unroll
                for (int d = 0; d < Op::ND; ++d)
                    if ((dm >> d) & 1u) part[d * Gv + vb] = acc[d];
            }
        }
    };
    if (rev) {  // no dot products: nothing to accumulate
        for (int st = 0; st < nrev; ++st) {
            const int jj = j++;
            const int slot = jj % NS;
            mbar_wait(&H->full[slot], (jj / NS) & 1);
            consume_tile(slot, (int)blockIdx.x + Gp * (nrev - 1 - st));
        }
    } else if (rr2) {
        // per-tile contributions (one term per dot per row) added into the
        // owning virtual CTA's accumulators in its tile order
        double acc0[Op::ND > 0 ? Op::ND : 1], acc1[Op::ND > 0 ? Op::ND : 1];
#pragma unroll
        for (int d = 0; d < Op::ND; ++d) acc0[d] = acc1[d] = 0.0;
        for (int st = 0;; ++st) {
            const int tile = rr2_tile(blockIdx.x, Gp, Gv, ntiles, st);
            if (tile == -2) break;
            if (tile < 0) continue;
            const int jj = j++;
            const int slot = jj % NS;
            mbar_wait(&H->full[slot], (jj / NS) & 1);
#pragma unroll
            for (int d = 0; d < Op::ND; ++d) acc[d] = 0.0;
            consume_tile(slot, tile);
            if (st & 1) {
#pragma unroll
                for (int d = 0; d < Op::ND; ++d) acc1[d] = ADD(acc1[d], acc[d]);
            } else {
#pragma unroll
                for (int d = 0; d < Op::ND; ++d) acc0[d] = ADD(acc0[d], acc[d]);
            }
        }
#pragma unroll
        for (int d = 0; d < Op::ND; ++d) acc[d] = acc0[d];
        close_vb(blockIdx.x);
#pragma unroll
        for (int d = 0; d < Op::ND; ++d) acc[d] = acc1[d];
        close_vb(blockIdx.x + Gp);
    } else {
        CGVK_FOR_VB(vb, P.order, blockIdx.x, Gv, Gp) {
#pragma unroll
            for (int d = 0; d < Op::ND; ++d) acc[d] = 0.0;
            CGVK_FOR_TILE(tile, P.order, vb, ntiles, Gv) {
                const int jj = j++;
                const int slot = jj % NS;
                mbar_wait(&H->full[slot], (jj / NS) & 1);
                if (jj == 0) tl_mark(Op::CSR, 2);
                consume_tile(slot, tile);
            }
            close_vb(vb);
        }
    }
    if (PdlLate<Op>::value) pdl_trigger();
    tl_mark(Op::CSR, 3);
    const int mode = op.sync();
    // chained: the next kernel finishes (single GPU: and folds the partials)
    if (mode == 0 || (chain && (mode == 1 || !PEER))) return;
    unsigned int* counter = op.counter(P);
    const bool is_last = arrive_last_c(counter, &H->last_flag);
    tl_mark(Op::CSR, 4);
    if (!is_last) return;
    double tot[Op::ND > 0 ? Op::ND : 1];
#pragma unroll
    for (int d = 0; d < Op::ND; ++d) tot[d] = 0.0;
    if (mode == 2) {
        if constexpr (Op::ND > 0) {
            fold_last<Op::ND>(P.part, Gv, t, H, stages, (size_t)NS * S.stage_bytes, tot);
            tl_mark(Op::CSR, 7);
            cta_tree_c<Op::ND>(tot, H->red);
        }
    }
    if (t == 0) *counter = 0u;
    if (PEER && chain) {  // the rank total; the next kernel folds the ranks and runs the scalar tail
        if (t == 0) p2p_publish_totals<Op::ND>(P.pp, H->cs.hseq, tot);
        tl_mark(Op::CSR, 6);
        return;
    }
    if (P.dist && mode == 2) {  // rank total: k_finalize folds all ranks in rank order
        if (t == 0) {
#pragma unroll
            for (int d = 0; d < Op::ND; ++d) P.rank_tot[d] = tot[d];
            if constexpr (HasDistMark<Op>::value) op.dist_mark(P, P.ctrl);
        }
        return;
    }
    tl_mark(Op::CSR, 5);
    finish_last(op, P, H, tot, t);
    tl_mark(Op::CSR, 6);
}

}  // namespace cgvk
