// Device-side building blocks shared by every cgvk kernel (sm_100a).
//
//  * Ctrl: the device-resident solver control block — SolverState's scalars
//    (inc/variants.hpp:122-130), status (:62-86), stats (:88-93) and the
//    fused-schedule bookkeeping. Written only by the single "last CTA" of a
//    reducing kernel (or, in the chained schedule, by CTA 0 of the next
//    kernel into the other of two copies); read by every CTA at kernel entry.
//  * The canonical reduction tree: one row per thread, per-
//    thread sequential sums over the tiles b, b+G, ..., a shfl_down warp tree,
//    a cross-warp tree, and a last-arriving-CTA final pass over the G CTA
//    partials. oracle/cgv_oracle.c (ORC_DOT_TREE) restates it bit-for-bit.
//  * Rounded arithmetic helpers: every multiply and add is rounded separately
//    (no FMA), as the reference is built with -ffp-contract=off
//    (proj/CMakeLists.txt:12-14). The whole library is also compiled with
//    --fmad=false.
#pragma once

#include <cstdint>

namespace cgvk {

constexpr int kBlock = 256;       // rows per tile == threads per CTA
constexpr int kWarps = kBlock / 32;
constexpr int kMinBlocksPerSM = 4;  // generic kernels: __launch_bounds__ minimum
constexpr int kVirtualPerSM = 12;   // canonical G cap = SMs * 12 (divisible by 2, 3, 4, 6 CTAs/SM)
constexpr int kVirtualPerSMCsr = 3;  // CSR engine: one virtual CTA per physical CTA (3 CTAs/SM)
constexpr int kVirtualPerSMBand = 6; // band engine (SpMV kernels 2 CTAs/SM, update kernels 3)
constexpr int kMaxDots = 6;

// SolverState scalar slots
enum { SA = 0, SB, SNU, SNUP, SMU, SDEL, SDELH, SGAM, SETA, NSCAL };
// status (inc/variants.hpp:62-86 order)
enum { ST_RUNNING = 0, ST_BREAKDOWN = 1, ST_MAXITER = 2, ST_CONVERGED = 3 };
enum { BR_NONE = 0, BR_NUPRIME, BR_NU, BR_MU, BR_NONFINITE };
enum { CB_ZERO = 0, CB_ERROR, CB_STAGNATION, CB_TOL };
// second-kernel modes
enum { MODE_SKIP = 0, MODE_FULL = 1, MODE_X_ONLY = 2 };
// stats slots
enum { STAT_SPMV = 0, STAT_BLOCK, STAT_PREC, STAT_RED };

struct __align__(16) Ctrl {
    double sc[NSCAL];
    double rr;     // <r,r> of the current r (canonical order)
    double tol;    // relative-residual stop (<= 0: off)
    double bnorm;  // ||b|| (canonical order)
    unsigned long long stats[4];
    int k;         // SolverState::k
    int k_limit;   // iterations run while k < k_limit
    int state, reason, criterion;
    int mode2;        // what the second kernel of the iteration must do
    int form_pending; // CG-CG / GV: the beta-recurrences of the last step are owed
    int pcur;         // HS: which p buffer is current
    int wt_stored;    // pipe-PR: w~ lives in its buffer (nu'-terminal step)
    int hist_cap;
    unsigned int count[2];  // last-CTA arrival counters
    int init_stage;         // initialize(): 0, or the check that settled the status (1 nu0, 2 mu0)
    // peer-memory exchange of a row-partitioned solve (cgvk_p2p.cuh): the
    // kernel sequence number (+1 per chained K1 / K2, identical on every
    // rank), and a GV / pipe-PR K1 reduction left to the next K1 (its stamp)
    unsigned int hseq;
    unsigned int defer;
    unsigned int dstamp;
    // spare (the chained schedule's successor folds the partials itself,
    // cgvk_stream.cuh chain_prologue); CTA 0 copies the words before it forward
    double tot[kMaxDots];
    double pad_[2];
};
static_assert(sizeof(Ctrl) == 256, "the control block is two 128-byte lines");

// Peer-memory exchange plan of one rank of a row-partitioned solve
// (cgvk_p2p.cuh): the rank's chained kernels push their boundary rows into
// the neighbours' receive buffers and their rank totals into every rank's
// table as stamped 8-byte words; consumers check the stamps as they read.
constexpr int kP2pSlots = 6;    // halo-exchanged vectors per variant (physical slots; PrF: 2 sets of 3)
constexpr int kP2pRanks = 8;    // ranks of one NVSwitch box
constexpr int kP2pTotSlots = 4; // rank-total tables in flight (by stamp & 3)

struct PeerPlan {
    int nranks, rank;
    int psel;               // HS: physical slots 1 / 2 = p0 / p1, p_old chosen by ctrl->pcur
    int tlo, hi_first;      // boundary tiles: [0, tlo) hold rows sent to the lower neighbour,
                            // [hi_first, ntiles) rows sent to the upper
    int nlo, hi0;           // send rows [0, nlo) -> lower neighbour, [hi0, n) -> upper
    int hbase;              // first halo column (local numbering)
    int rx_stride;          // receive entries per parity: nlow + nup
    int lo_off, lo_stride;  // lower neighbour: where my rows land in its buffer (its nlow), its stride
    int hi_stride;          // upper neighbour's stride (my rows land at its 0)
    double* hv[kP2pSlots];                  // this rank's halo-exchanged vectors (physical slots)
    unsigned long long* rx[kP2pSlots];      // mine: [2 parities][rx_stride] entries of 2 words
    unsigned long long* rx_lo[kP2pSlots];   // the lower neighbour's receive buffers (null: none)
    unsigned long long* rx_hi[kP2pSlots];   // the upper neighbour's
    unsigned int* err;      // set when a wait gives up
    long long delay_ns;     // experiments (CGVK_P2P_DELAY_NS): a published total counts as
                            // arrived only this long after its publication (an injected
                            // link latency; 0: off)
    double* xtot_peer[kP2pRanks];  // every rank's total tables
};

struct Params {
    int n, ntiles;
    const int* __restrict__ rp;
    const int* __restrict__ ci;
    const double* __restrict__ va;
    const double* __restrict__ d;  // Jacobi inv_diag (PREC) or null
    double* x;
    double* r;
    double* p0;
    double* p1;
    double* s;
    double* w;
    double* u;
    double* t;
    double* rt;
    double* st;
    double* wt;
    double* wpred;  // run() with probes: pipe-PR's predicted w'_k (src/variants.cpp:312), or null
    double *b0, *b1, *b2;  // one kernel per iteration: second buffers (GvF: w, u, t; PprF: s~ | s, r~ | r, w)
    // band engine (cgvk_band.cuh): SELL-C-sigma copy of A, null when unused
    const int* __restrict__ band_off;             // slice offsets (entries), ntiles*8+1
    const unsigned int* __restrict__ band_meta;   // per tile slot: len << 8 | tile-local row
    const double* __restrict__ band_va;
    const unsigned short* __restrict__ band_ci;   // column - (tile - band_h) * 256
    int band_h;                                   // window half-width in tiles
    double* part;  // [kMaxDots][G] CTA partials
    double* part_b;  // chained schedule: K1's partials (K2 writes `part`)
    double* hist;  // rr per iteration (null: not recorded by this CTA)
    Ctrl* ctrl;
    // chained schedule (cgvk_stream.cuh chain_prologue): the second control
    // block (K1 writes ctrl_b, K2 writes ctrl)
    Ctrl* ctrl_b;
    int nu_expr, recompute_nu, recompute_w, unsimplified_mu, track_delta;
    int order;  // canonical tile order (see CGVK_FOR_VB)
    int l2pol;  // TMA L2 policy: 0 evict_first everything, 1 only the matrix, 2 none
    int dist;          // rank of a row-partitioned solve: reducing kernels stop at the
    double* rank_tot;  // rank-local totals [kMaxDots]; k_finalize folds all ranks
    const PeerPlan* pp;  // chained rank kernels exchanging through peer memory (device copy; null: off)
};

// Balanced contiguous partition: part k of `parts` covers [lo(k), lo(k+1)).
// Canonical order: virtual CTA vb owns tiles [lo(vb; ntiles, Gv), lo(vb+1));
// a physical CTA p runs virtual CTAs [lo(p; Gv, Gp), lo(p+1)) — neighbouring
// rows stay on one SM, so stencil x-gathers hit L1.
__host__ __device__ __forceinline__ int span_lo(int k, int total, int parts) {
    return static_cast<int>(static_cast<long long>(k) * total / parts);
}

// Tile orders (the oracle's orc_dotcfg.order): 0 strided — virtual CTA vb
// owns tiles vb, vb+Gv, ..., physical CTA p runs vb = p, p+Gp, ...; 1
// contiguous — the span_lo blocks above.
#define CGVK_FOR_VB(vb, order, p, Gv, Gp)                                              \
    for (int vb = (order) ? span_lo((p), (Gv), (Gp)) : (p),                            \
             vb##_end = (order) ? span_lo((p) + 1, (Gv), (Gp)) : (Gv),                  \
             vb##_step = (order) ? 1 : (Gp);                                            \
         vb < vb##_end; vb += vb##_step)
#define CGVK_FOR_TILE(tile, order, vb, ntiles, Gv)                                     \
    for (int tile = (order) ? span_lo((vb), (ntiles), (Gv)) : (vb),                    \
             tile##_end = (order) ? span_lo((vb) + 1, (ntiles), (Gv)) : (ntiles),       \
             tile##_step = (order) ? 1 : (Gv);                                          \
         tile < tile##_end; tile += tile##_step)

__device__ __forceinline__ double MUL(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ADD(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double SUB(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double DIV(double a, double b) { return __ddiv_rn(a, b); }

// Canonical CTA tree over ND per-thread values; the totals end up in thread 0.
template <int ND>
__device__ __forceinline__ void cta_tree(double (&v)[ND], double* sm /* ND*32 */) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int d = 0; d < ND; ++d) {
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1)
            v[d] = ADD(v[d], __shfl_down_sync(0xffffffffu, v[d], off));
    }
    if (lane == 0) {
#pragma unroll
        for (int d = 0; d < ND; ++d) sm[d * 32 + warp] = v[d];
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int d = 0; d < ND; ++d) {
            double y = lane < kWarps ? sm[d * 32 + lane] : 0.0;
#pragma unroll
            for (int off = kWarps / 2; off >= 1; off >>= 1)
                y = ADD(y, __shfl_down_sync(0xffffffffu, y, off));
            v[d] = y;
        }
    }
    __syncthreads();
}

// Arrive on `counter`; true in every thread of the last CTA to arrive.
__device__ __forceinline__ bool arrive_last(unsigned int* counter) {
    __shared__ int last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned int prev = atomicAdd(counter, 1u);
        last = prev == gridDim.x - 1;
    }
    __syncthreads();
    if (last) __threadfence();
    return last != 0;
}

// Write this CTA's ND partials, arrive, and (last CTA only) fold all G
// partials into tot[] (valid in thread 0). Returns true in the last CTA.
template <int ND>
__device__ __forceinline__ bool reduce_grid(double (&acc)[ND], double* part, unsigned int* counter,
                                            double (&tot)[ND]) {
    __shared__ double sm[ND * 32];
    cta_tree<ND>(acc, sm);
    const int G = gridDim.x;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int d = 0; d < ND; ++d) part[d * G + blockIdx.x] = acc[d];
    }
    if (!arrive_last(counter)) return false;
#pragma unroll
    for (int d = 0; d < ND; ++d) tot[d] = 0.0;
    for (int j = threadIdx.x; j < G; j += kBlock) {
#pragma unroll
        for (int d = 0; d < ND; ++d) tot[d] = ADD(tot[d], __ldcg(part + d * G + j));
    }
    cta_tree<ND>(tot, sm);
    if (threadIdx.x == 0) *counter = 0u;
    return true;
}

// ------------------------------------------------ status helpers (thread 0)
// src/variants.cpp:128-173

__device__ __forceinline__ void fail(Ctrl* c, int reason) {
    c->state = ST_BREAKDOWN;
    c->reason = reason;
}

// settle_nonpositive; rr = <r,r> of the current r (an exact-zero test, so the
// summation order cannot change the outcome)
__device__ __forceinline__ bool settle_nonpositive(Ctrl* c, double value, int reason, double rr) {
    if (!isfinite(value)) {
        fail(c, BR_NONFINITE);
        return true;
    }
    if (value > 0.0) return false;
    if (value == 0.0 && rr == 0.0) {
        c->state = ST_CONVERGED;
        c->criterion = CB_ZERO;
    } else {
        fail(c, reason);
    }
    return true;
}

__device__ __forceinline__ bool settle_mu(Ctrl* c) {
    const double mu = c->sc[SMU];
    if (!isfinite(mu)) {
        fail(c, BR_NONFINITE);
        return true;
    }
    if (mu <= 0.0) {
        fail(c, BR_MU);
        return true;
    }
    return false;
}

__device__ __forceinline__ bool finalize_alpha(Ctrl* c) {
    c->sc[SA] = DIV(c->sc[SNU], c->sc[SMU]);
    if (!isfinite(c->sc[SA]) || !isfinite(c->sc[SB])) {
        fail(c, BR_NONFINITE);
        return true;
    }
    return false;
}

// predicted_nu, src/variants.cpp:175-187; operands are the k-1 values
__device__ __forceinline__ double predicted_nu(int expr, const double* sc) {
    const double a = sc[SA];
    const double a2g = MUL(MUL(a, a), sc[SGAM]);
    if (expr == 1) return ADD(SUB(sc[SNU], MUL(MUL(2.0, a), sc[SDEL])), a2g);   // Simplified
    if (expr == 2) return ADD(-sc[SNU], a2g);                                  // Meurant
    return ADD(SUB(sc[SNU], MUL(a, ADD(sc[SDEL], sc[SDELH]))), a2g);           // Expanded
}

// Harness stop rule ||r_k|| <= tol*||b||, checked after a step.
__device__ __forceinline__ void check_tolerance(Ctrl* c) {
    if (c->state == ST_RUNNING && c->tol > 0.0 && sqrt(c->rr) <= MUL(c->tol, c->bnorm)) {
        c->state = ST_CONVERGED;
        c->criterion = CB_TOL;
    }
}

__device__ __forceinline__ void record_rr(const Params& P, Ctrl* c, double rr) {
    c->rr = rr;
    if (P.hist && c->k < c->hist_cap) P.hist[c->k] = rr;
}

// CSR row product, left-to-right, each term rounded (sparse_matrix.cpp:112-117).
template <class XF>
__device__ __forceinline__ double row_sum(const Params& P, int row, XF xf) {
    const int k0 = __ldg(P.rp + row), k1 = __ldg(P.rp + row + 1);
    double sum = 0.0;
#pragma unroll 4
    for (int k = k0; k < k1; ++k) sum = ADD(sum, MUL(__ldg(P.va + k), xf(__ldg(P.ci + k))));
    return sum;
}

// two right-hand sides in one traversal (sparse_matrix.cpp:131-142)
template <class XF1, class XF2>
__device__ __forceinline__ void row_sum2(const Params& P, int row, XF1 xf1, XF2 xf2, double& y1,
                                         double& y2) {
    const int k0 = __ldg(P.rp + row), k1 = __ldg(P.rp + row + 1);
    double s1 = 0.0, s2 = 0.0;
#pragma unroll 4
    for (int k = k0; k < k1; ++k) {
        const double v = __ldg(P.va + k);
        const int c = __ldg(P.ci + k);
        s1 = ADD(s1, MUL(v, xf1(c)));
        s2 = ADD(s2, MUL(v, xf2(c)));
    }
    y1 = s1;
    y2 = s2;
}

}  // namespace cgvk
