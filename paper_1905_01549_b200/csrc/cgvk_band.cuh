// Band engine: the SpMV kernels (K2 of every variant) for matrices whose
// columns stay within a narrow band around the diagonal and whose rows are
// long (R4M: ~27 entries/row within +-4096), where gathering x through L1
// costs one L1 tag lookup per entry and the SM's L1 pipeline, not HBM, sets
// the kernel time (profiles/r01: 72 % L1 throughput, 3.2 TB/s DRAM).
//
// Matrix layout (built once, cgvk_api.cu build_band): SELL-C-sigma with C = 32
// and sigma = 256 — inside each 256-row tile the rows are sorted by length
// (descending, stable) and dealt to the 8 warps as 32-row slices; entry k of a
// slice's rows is stored interleaved (va[32 k + lane]), so every matrix load
// is one coalesced warp access and a slice is padded only to its own longest
// row. Columns are 16-bit offsets from the tile's window base (tile - H) * 256
// (10 B/entry instead of 12). Per tile slot: meta = len << 8 | tile-local row.
//
// Per CTA (288 threads: 8 consumer warps + a producer warp, tiles in the
// contiguous canonical order): the producer keeps, for each gathered operand,
// a ring of 2H + NS tiles of that vector in shared memory — the window
// [tile - H, tile + H] of the tile being computed plus the lookahead — adding
// one 2 KB tile per step with a bulk copy, together with the tile's meta,
// slice offsets and staged per-row vectors, and prefetches the tile's slice
// data into L2 (cp.async.bulk.prefetch) a few tiles ahead. Consumers read
// their slice straight from L2 and gather x from the window (shared memory).
//
// Bits: a row's sum is still left to right over its CSR entries; the per-row
// dot contributions are written to shared memory at the row's tile-local
// position and added in the canonical order (thread t <- row t), so the
// reductions are exactly those of the CSR pipeline with order 1.
#pragma once

#include "cgvk_stream.cuh"

namespace cgvk {

constexpr int kBandMetaBytes = kBlock * 4;     // meta words
constexpr int kBandOffBytes = 64;              // 9 slice offsets (+ pad)
constexpr int kBandMaxNG = 2;

__host__ __device__ inline int band_stage_bytes(int nvec) {
    return (kBandMetaBytes + kBandOffBytes + nvec * kBlock * 8 + 127) & ~127;
}

struct BandIn {
    const double* sv;   // stage vectors + tile-local row
    const double* w0;   // window rings of the gathered operands
    const double* w1;
    __device__ __forceinline__ double operator()(int v) const { return sv[v * kBlock]; }
    __device__ __forceinline__ double gather(int k, int q, const double*) const { return (k ? w1 : w0)[q]; }
    // transform window (BAND_XF): ring 0 already holds the combined operand
    __device__ __forceinline__ double gather_p(int q, const double*, const double*, double) const { return w0[q]; }
};

// Windows a band kernel keeps (one when the Op combines its sources) and the
// raw source tiles each stage carries for the consumers to combine.
// Two-window kernels run one CTA per SM; those without dot products (pipe-PR's
// block SpMV) then use two consumer groups of 8 warps that take alternate
// tiles, for twice the loads in flight.
template <class Op>
struct BandShape {
    static constexpr bool XF = BandXf<Op>::value;
    static constexpr int NWIN = XF ? 1 : Op::NG;
    static constexpr int NRAW = XF ? Op::NG : 0;
    static constexpr int GROUPS = (NWIN == 2 && Op::ND == 0) ? 2 : 1;
    static constexpr int THREADS = GROUPS * kBlock + 32;
    static constexpr int MINB = NWIN == 2 ? 1 : 2;
};

template <int N>
__device__ __forceinline__ void named_sync1() {
    asm volatile("bar.sync 1, %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// Entries per chunk of the row product: the two-operand kernels run one CTA
// per SM (two window rings), so they get the registers for longer chunks.
#ifndef CGVK_BAND_CHUNK
#define CGVK_BAND_CHUNK 8
#endif
#ifndef CGVK_BAND_CHUNK2
#define CGVK_BAND_CHUNK2 8
#endif

// Register cap of the two-CTA band kernels with dot products: __maxnreg__
// instead of __launch_bounds__(288, 2), under which ptxas settles at 95-96
// registers. Measured on R4M: 104 registers, still two CTAs per
// SM, HS 353 -> 342 us, CG 357 -> 353, M/PR 359 -> 352; GV's dot-free K2
// keeps the launch bounds (395 vs 390 us with the cap). make_band takes the
// capped form only where it keeps two CTAs per SM. 0 = launch bounds.
#ifndef CGVK_BAND_MAXNREG
#define CGVK_BAND_MAXNREG 104
#endif
// Kernels with dot products: 1 = warps rotate over the slices and hand the
// per-row contributions over through two mbarrier-guarded buffers, folding
// tile k's while computing tile k+1 (a warp may run one tile ahead of the
// slowest); 0 = one CTA barrier per tile, fixed slices (round 1).
#ifndef CGVK_BAND_SLACK
#define CGVK_BAND_SLACK 1
#endif
// tiles between a combined window tile (BAND_XF) and its first reader
constexpr int kBandXfAhead = 1 + CGVK_BAND_SLACK;
template <class Op, class Prev>
__device__ __forceinline__ void band_body(const Params& P, const StageCfg& S);

template <class Op, class Prev>
__global__ void __launch_bounds__(BandShape<Op>::THREADS, BandShape<Op>::MINB) k_band(Params P, StageCfg S) {
    band_body<Op, Prev>(P, S);
}
#if CGVK_BAND_MAXNREG
template <class Op, class Prev>
__global__ void __maxnreg__(CGVK_BAND_MAXNREG) k_band_nr(Params P, StageCfg S) {
    band_body<Op, Prev>(P, S);
}
#endif

template <class Op, class Prev>
__device__ __forceinline__ void band_body(const Params& P, const StageCfg& S) {
    static_assert(Op::CSR && Op::NG <= kBandMaxNG, "band engine runs the SpMV kernels");
    using Shape = BandShape<Op>;
    constexpr bool XF = Shape::XF;
    constexpr int NWIN = Shape::NWIN;
    constexpr int GR = Shape::GROUPS;
    constexpr int NC = GR * kConsumers;  // consumer threads
    static_assert(!XF || Op::ND > 0, "a combined window relies on the contribution hand-over for ordering");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    PipeHeader* H = reinterpret_cast<PipeHeader*>(smem_raw);
    unsigned char* stages = smem_raw + ((sizeof(PipeHeader) + 127) / 128) * 128;
    const int NS = S.nstage, RT = S.ring, RW = RT * kBlock, HB = P.band_h;
    double* win = reinterpret_cast<double*>(stages + (size_t)NS * S.stage_bytes);
    double* cbuf = win + (size_t)NWIN * RW;
    const int Gv = S.gvirt, Gp = gridDim.x, ntiles = P.ntiles;
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(&H->full[s], 1);
            mbar_init(&H->empty[s], kWarps);
        }
        mbar_init(&H->fold_bar, 1);
        for (int b = 0; b < 2; ++b) {
            mbar_init(&H->cfull[b], kWarps);
            mbar_init(&H->cempty[b], kWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    pdl_wait();
    pdl_trigger();
    const int chain = S.chain;
    if (chain) chain_prologue<Op, Prev>(P, chain, H, (chain & CH_ODD) ? P.ctrl : P.ctrl_b, S.gprev);
    double* const partw = (chain && !(chain & CH_ODD)) ? P.part_b : P.part;
    Op op;
    if (!(chain ? op.enter(with_ctrl(P, &H->cs)) : op.enter(P))) return;  // uniform over the grid

    // this CTA's contiguous run of tiles (order 1)
    const int vb0 = span_lo(blockIdx.x, Gv, Gp), vb1 = span_lo(blockIdx.x + 1, Gv, Gp);
    const int T0 = span_lo(vb0, ntiles, Gv), T1 = span_lo(vb1, ntiles, Gv);

    if (warp == GR * kWarps) {  // ------------------------- producer warp
        if (threadIdx.x != NC) return;
        const uint64_t vpol = P.l2pol == 0 ? evict_first_policy() : 0;
        const double* vp[kMaxVec];
#pragma unroll
        for (int v = 0; v < Op::NV; ++v) vp[v] = op.vec(P, v);
        const double* gp[kBandMaxNG] = {nullptr, nullptr};
#pragma unroll
        for (int k = 0; k < Op::NG; ++k) gp[k] = op.gsrc(P, k);
        auto tile_bytes = [&](int u) -> uint32_t { return (min(kBlock, P.n - u * kBlock) * 8 + 15) & ~15; };
        auto prefetch = [&](int u) {
            if (u >= T1) return;
            const int e0 = __ldg(P.band_off + u * kWarps), e1 = __ldg(P.band_off + u * kWarps + kWarps);
            if (e1 > e0) {
                bulk_prefetch_l2(P.band_va + e0, (uint32_t)(e1 - e0) * 8u);
                bulk_prefetch_l2(P.band_ci + e0, (uint32_t)(e1 - e0) * 2u);
            }
        };
        for (int u = T0; u < T0 + S.pf && u < T1; ++u) prefetch(u);
        const int w_lo = max(0, T0 - HB), w_hi = min(ntiles, T0 + HB);  // prologue window tiles
        for (int t = T0; t < T1; ++t) {
            const int j = t - T0, slot = j % NS;
            if (j >= NS) mbar_wait(&H->empty[slot], ((j / NS) - 1) & 1);
            unsigned char* st = stages + (size_t)slot * S.stage_bytes;
            double* sv = reinterpret_cast<double*>(st + kBandMetaBytes + kBandOffBytes);
            const int r0 = t * kBlock;
            const uint32_t vb = tile_bytes(t);
            // window tile entering the ring: t + H (raw windows, straight into
            // the ring) or t + H + kBandXfAhead (XF: staged raw, combined by
            // the consumers that many tiles before its first reader)
            const int u = XF ? t + HB + kBandXfAhead : t + HB;
            uint32_t bytes = kBandMetaBytes + 48;
#pragma unroll
            for (int v = 0; v < Op::NV; ++v)
                if (vp[v]) bytes += vb;
#pragma unroll
            for (int k = 0; k < Op::NG; ++k)
                if (gp[k] && u < ntiles) bytes += tile_bytes(u);
            if (!XF && j == 0) {
                for (int q = w_lo; q < w_hi; ++q)
#pragma unroll
                    for (int k = 0; k < Op::NG; ++k)
                        if (gp[k]) bytes += tile_bytes(q);
            }
            mbar_expect_tx(&H->full[slot], bytes);
            bulk_g2s(st, P.band_meta + (size_t)t * kBlock, kBandMetaBytes, &H->full[slot], 0);
            bulk_g2s(st + kBandMetaBytes, P.band_off + (size_t)t * kWarps, 48, &H->full[slot], 0);
#pragma unroll
            for (int v = 0; v < Op::NV; ++v)
                if (vp[v]) bulk_g2s(sv + v * kBlock, vp[v] + r0, vb, &H->full[slot], vpol);
            auto load_win = [&](int q) {
#pragma unroll
                for (int k = 0; k < Op::NG; ++k)
                    if (gp[k])
                        bulk_g2s(win + (size_t)k * RW + (q % RT) * kBlock, gp[k] + (size_t)q * kBlock,
                                 tile_bytes(q), &H->full[slot], 0);
            };
            if constexpr (XF) {
                if (u < ntiles)
#pragma unroll
                    for (int k = 0; k < Op::NG; ++k)
                        bulk_g2s(sv + (Op::NV + k) * kBlock, gp[k] + (size_t)u * kBlock, tile_bytes(u),
                                 &H->full[slot], 0);
            } else {
                if (j == 0)
                    for (int q = w_lo; q < w_hi; ++q) load_win(q);
                if (u < ntiles) load_win(u);
            }
            prefetch(t + S.pf);
        }
        return;
    }

    // ------------------------------------------------------ consumer warps
    //
    // Slices of a tile are sorted by row length, so slice 0 is the longest
    // (R4M: its longest row averages 38 entries against a 28-entry mean over
    // the slices). Kernels without dot products have no per-tile barrier:
    // their warps rotate over the slices (warp w takes slice (w + tile) % 8),
    // so every warp does the same work over any 8 tiles and the stage ring
    // absorbs the drift (measured R4M: GV K2 283 -> 265 us, pipe-PR K2 313 ->
    // 284 us). Kernels with dot products exchange the per-row contributions
    // through shared memory after every tile (one CTA barrier), so there the
    // longest slice sets each tile's time whatever the map; taking tiles in
    // pairs with balanced slices measured 1.6-2.2x slower (register spills and
    // a second copy of the row loop), see DESIGN.md §9.
    const int t = threadIdx.x & (kBlock - 1), lane = t & 31, grp = threadIdx.x / kBlock;
    const int wg = warp & (kWarps - 1);  // warp within its group
    if constexpr (XF) {
        // prologue: the window [T0 - H, T0 + H] of the first tile, combined
        // from global (later tiles get theirs from the stages)
        const double* g0 = op.gsrc(P, 0);
        const double* g1 = op.gsrc(P, 1);
        const int q0 = max(0, T0 - HB) * kBlock, q1 = min(P.n, (T0 + HB + kBandXfAhead) * kBlock);
        for (int q = q0 + t; q < q1; q += kConsumers)
            win[(q / kBlock) % RT * kBlock + q % kBlock] = op.band_xf(__ldg(g0 + q), __ldg(g1 + q));
        consumer_sync();
    }
    double acc[Op::ND > 0 ? Op::ND : 1];
    int j = 0;
    // thread t adds row t's contribution of the CTA's tile x (x = tile - T0)
    // to its accumulators, in tile order, once every warp has written it
    auto fold_tile = [&](int x) {
        if constexpr (Op::ND > 0) {
            const double* cb = cbuf + (x & 1) * (Op::ND * kBlock);
            mbar_wait(&H->cfull[x & 1], (x >> 1) & 1);
            if ((T0 + x) * kBlock + t < P.n) {
#pragma unroll
                for (int d = 0; d < Op::ND; ++d) acc[d] = ADD(acc[d], cb[d * kBlock + t]);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&H->cempty[x & 1]);
        }
    };
    for (int vb = vb0; vb < vb1; ++vb) {
        const int jv = j;  // the virtual CTA's first tile (CTA-relative)
#pragma unroll
        for (int d = 0; d < Op::ND; ++d) acc[d] = 0.0;
        const int te = span_lo(vb + 1, ntiles, Gv);
        for (int tile = span_lo(vb, ntiles, Gv); tile < te; ++tile) {
            const int jj = j++;
            if (GR > 1 && jj % GR != grp) continue;  // the other group's tile
            const int slot = jj % NS;
            mbar_wait(&H->full[slot], (jj / NS) & 1);
            const unsigned char* st = stages + (size_t)slot * S.stage_bytes;
            const double* sv = reinterpret_cast<const double*>(st + kBandMetaBytes + kBandOffBytes);
            if constexpr (XF) {  // combine window tile tile + H + kBandXfAhead
                const int u = tile + HB + kBandXfAhead;
                if (u < ntiles && u * kBlock + t < P.n)
                    win[(u % RT) * kBlock + t] = op.band_xf(sv[Op::NV * kBlock + t], sv[(Op::NV + 1) * kBlock + t]);
            }
            const int slice = (Op::ND > 0 && !CGVK_BAND_SLACK) ? wg : (wg + jj / GR) & (kWarps - 1);
            const unsigned int meta = reinterpret_cast<const unsigned int*>(st)[slice * 32 + lane];
            const int rl = meta & 255;
            const int off = reinterpret_cast<const int*>(st + kBandMetaBytes)[slice];
            const int r0 = tile * kBlock;
            const int i = r0 + rl;
            double tmp[Op::ND > 0 ? Op::ND : 1];
#pragma unroll
            for (int d = 0; d < Op::ND; ++d) tmp[d] = 0.0;
            if (i < P.n) {
                int tb = (tile - HB) % RT;
                if (tb < 0) tb += RT;
                const BandRow<NWIN == 2 ? CGVK_BAND_CHUNK2 : CGVK_BAND_CHUNK> R{
                    P.band_va + off + lane, P.band_ci + off + lane, static_cast<int>(meta >> 8), tb * kBlock, RW};
                op.row(P, i, BandIn{sv + rl, win, win + RW}, R, tmp);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&H->empty[slot]);
            if constexpr (Op::ND > 0) {
                // per-row contributions back to canonical positions
                double* cb = cbuf + (jj & 1) * (Op::ND * kBlock);
                if (CGVK_BAND_SLACK && jj >= 2) mbar_wait(&H->cempty[jj & 1], ((jj >> 1) - 1) & 1);
#pragma unroll
                for (int d = 0; d < Op::ND; ++d) cb[d * kBlock + rl] = tmp[d];
                if (CGVK_BAND_SLACK) {
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&H->cfull[jj & 1]);
                    if (jj > jv) fold_tile(jj - 1);  // the previous tile, now complete
                } else {
                    consumer_sync();
                    if (r0 + t < P.n) {
#pragma unroll
                        for (int d = 0; d < Op::ND; ++d) acc[d] = ADD(acc[d], cb[d * kBlock + t]);
                    }
                }
            }
        }
        if constexpr (Op::ND > 0) {
            if (CGVK_BAND_SLACK && j > jv) fold_tile(j - 1);  // the virtual CTA's last tile
            if (op.sync() != 2) continue;
            cta_tree_c<Op::ND>(acc, H->red);
            if (t == 0) {
#pragma unroll
                for (int d = 0; d < Op::ND; ++d) partw[d * Gv + vb] = acc[d];
            }
        }
    }
    const int mode = op.sync();
    // chained: the next kernel finishes (and folds the partials)
    if (mode == 0 || chain) return;
    unsigned int* counter = op.counter(P);
    if constexpr (GR > 1) {  // no dots: arrive, the last CTA finishes
        static_assert(GR == 1 || Op::ND == 0, "consumer groups only without dot products");
        named_sync1<NC>();
        if (threadIdx.x == 0) {
            __threadfence();
            H->last_flag = atomicAdd(counter, 1u) == gridDim.x - 1;
        }
        named_sync1<NC>();
        if (!H->last_flag || threadIdx.x != 0) return;
        __threadfence();
        *counter = 0u;
        const double none[1] = {0.0};
        op.finish(P, P.ctrl, none);
        return;
    }
    if (!arrive_last_c(counter, &H->last_flag)) return;
    double tot[Op::ND > 0 ? Op::ND : 1];
#pragma unroll
    for (int d = 0; d < Op::ND; ++d) tot[d] = 0.0;
    if (mode == 2) {
        if constexpr (Op::ND > 0) {
            // the idle stage ring and window rings hold the partials
            fold_last<Op::ND>(P.part, Gv, t, H, stages, (size_t)NS * S.stage_bytes + (size_t)NWIN * RW * 8, tot);
            cta_tree_c<Op::ND>(tot, H->red);
        }
    }
    if (t == 0) *counter = 0u;
    if (P.dist && mode == 2) {
        if (t == 0) {
#pragma unroll
            for (int d = 0; d < Op::ND; ++d) P.rank_tot[d] = tot[d];
            if constexpr (HasDistMark<Op>::value) op.dist_mark(P, P.ctrl);
        }
        return;
    }
    finish_last(op, P, H, tot, t);
}

}  // namespace cgvk
