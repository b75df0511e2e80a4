// The per-iteration kernels of the six CG variants (+ pipe-PR-M; M-CG is the
// PR stepper with the Meurant nu'), as fused two-kernel schedules (SURVEY.md
// Appendix A), each an "Op" run by the TMA-staged pipeline of
// cgvk_stream.cuh.
//
// Each iteration is two launches, K1 then K2, captured in a CUDA graph — or,
// for problems that fit L2, ONE launch doing both halves (PrF, CgF, GvF, PprF
// below: the SpMV operand re-formed at every gathered column, same bits).
// Global reductions are folded by the next kernel's prologue (chained graphs)
// or the last-arriving CTA of the kernel that produces the operands, which
// also runs the scalar recurrences and the breakdown/convergence checks of
// src/variants.cpp:128-187 on the device, so the host never synchronises
// inside the loop. Every vector value is bit-
// identical to the reference's (no FMA; the Jacobi products d∘v that the
// reference stores are recomputed on the fly from the same operands); dots
// follow the canonical tree of cgvk_device.cuh.
//
// After K1/K2 of step k the device holds the reference state after step(k)
// (src/variants.cpp:446-458) except for the beta-recurrences that CG-CG and GV
// defer into the next K1 (`form_pending`); the host materialises them (a K1
// launch with k_limit = k) before reading vectors. Terminal steps keep the
// reference's partial-update semantics through `mode2` / `form_pending`.
//
// Staged per-row vectors are read as in(v); SpMV operands are gathered by
// column as in.gather(k, j, g): operand k (0 <= k < NG, source gsrc(P, k)),
// from global memory g (L1/L2) or from the band engine's shared-memory window.
#pragma once

#include "cgvk_stream.cuh"

namespace cgvk {

#ifndef CGVK_HS_LATE
#define CGVK_HS_LATE 3  // HS K1 (1) / K2 (2) signal their dependents after their tiles
#endif
#ifndef CGVK_K1_MAXNREG
#define CGVK_K1_MAXNREG 72  // GV / pipe-PR K1 under __maxnreg__ when the working set fits L2
#endif
#ifndef CGVK_SPMV_MAXNREG
#define CGVK_SPMV_MAXNREG 0  // > 0: the CSR SpMV kernels under __maxnreg__ (A/B)
#endif
#ifndef CGVK_CG_LATE
#define CGVK_CG_LATE 2  // CG-CG K1 (1) / K2 (2) signal their dependents after their tiles
#endif
#ifndef CGVK_GV_LATE
#define CGVK_GV_LATE 3  // GV K1 (1) / K2 (2) signal their dependents after their tiles
#endif
#ifndef CGVK_PPR_LATE
#define CGVK_PPR_LATE 2  // pipe-PR K1 (1) / K2 (2) signal their dependents after their tiles
#endif
#ifndef CGVK_PRF_LATE
#define CGVK_PRF_LATE 0  // the one-kernel PR / M iteration signals its dependent after its tiles
#endif
#ifndef CGVK_F_LATE
#define CGVK_F_LATE 0  // CgF (1) / GvF (2) / PprF (4) signal their dependent after their tiles
#endif
#ifndef CGVK_PRF_EARLY
#define CGVK_PRF_EARLY 1  // first stages' vectors issued right after the wait
#endif
#if CGVK_PRF_EARLY
#define CGVK_PRF_EVEC early_vec
#else
#define CGVK_PRF_EVEC evec_off
#endif
#ifndef CGVK_GV_K1_CTAS
#define CGVK_GV_K1_CTAS 3  // stage ring sized for this many resident CTAs (registers allow 2)
#endif
#ifndef CGVK_PPR_K1_CTAS
#define CGVK_PPR_K1_CTAS 3
#endif

template <bool PREC>
__device__ __forceinline__ double Mg(const Params& P, int j, double v) {  // gathered d_j * v
    if constexpr (PREC) return MUL(__ldg(P.d + j), v);
    return v;
}

__device__ __forceinline__ bool step_wanted(const Ctrl* c) {
    return c->state == ST_RUNNING && c->k < c->k_limit;
}

#define SV(v) in(v)

// Outputs that the next kernel does not read: streaming stores (L2
// evict-first), so they leave L2 to the vectors it does read — when the
// working set exceeds L2 (l2pol != 3; a problem that fits keeps everything).
// Measured P128: GV 92.7 -> 88.2 us, pipe-PR 84.2 -> 80.7 us;
// V256 neutral. CGVK_K1_STCS=0: plain stores (A/B).
#ifndef CGVK_K1_STCS
#define CGVK_K1_STCS 1
#endif
__device__ __forceinline__ void st_far(const Params& P, double* p, double v) {
#if CGVK_K1_STCS
    if (P.l2pol != 3) {
        __stcs(p, v);
        return;
    }
#endif
    *p = v;
}

// =====================================================================  HS
// src/variants.cpp:189-205, paper Alg. 1. V = 3+1 (K1) + 4+3 (K2) vectors.

// K1: r -= alpha*s; nu = <M r, r>, <r,r>.   streams: r s [d]
template <bool PREC>
struct HsK1 {
    static constexpr int NV = PREC ? 3 : 2, ND = 2;
    static constexpr bool CSR = false;
    static constexpr bool PDL_LATE = (CGVK_HS_LATE & 1) != 0;  // see cgvk_stream.cuh PdlLate
    double alpha;
    __device__ bool enter(const Params& P) {
        if (!step_wanted(P.ctrl)) return false;
        alpha = P.ctrl->sc[SA];
        return true;
    }
    // early_vec: the first stages issued right after the wait. Measured with
    // the successor fold: P64 HS 14.8 -> 14.5 us, P2D 10.7 ->
    // 10.5, P128 neutral (before it, with the last-CTA fold: P128 68.0 -> 69.1)
    __device__ const double* vec(const Params& P, int v) const { return early_vec(P, v); }
    __device__ static const double* early_vec(const Params& P, int v) { return v == 0 ? P.r : v == 1 ? P.s : P.d; }
    __device__ int sync() const { return 2; }
    __device__ unsigned int* counter(const Params& P) const { return &P.ctrl->count[0]; }
    template <class In, class RR>
    __device__ void row(const Params& P, int i, const In& in, const RR&, double* acc) const {
        const double r = SUB(SV(0), MUL(alpha, SV(1)));
        if (PREC) st_far(P, P.r + i, r);  // K2 reads r~ (without Jacobi it gathers r)
        else P.r[i] = r;
        double rt = r;
        if constexpr (PREC) {  // r~ = M r stored for K2 (its gather and own-row read)
            rt = MUL(SV(2), r);
            P.rt[i] = rt;
        }
        acc[0] = ADD(acc[0], MUL(rt, r));
        acc[1] = ADD(acc[1], MUL(r, r));
    }
    __device__ void finish(const Params& P, Ctrl* c, const double* tot) const {
        c->k += 1;
        c->stats[STAT_PREC] += PREC;
        c->stats[STAT_RED] += 1;
        record_rr(P, c, tot[1]);
        const double nu_next = tot[0];
        if (settle_nonpositive(c, nu_next, BR_NU, tot[1])) {
            c->sc[SNU] = nu_next;
            c->mode2 = MODE_X_ONLY;  // x_k = x_{k-1} + alpha p_{k-1} still owed
            return;
        }
        c->sc[SB] = DIV(nu_next, c->sc[SNU]);
        c->sc[SNU] = nu_next;
        c->mode2 = MODE_FULL;
    }
};

// K2: x += alpha*p_old; p = r~ + beta p_old (on the fly for every gathered
// column; r~ = M r stored by K1); s = A p; mu = <p,s>.   streams: A, p_old r~ x
template <bool PREC>
struct HsK2 {
    static constexpr int NV = 3, ND = 1;
    static constexpr int MAXNREG = CGVK_SPMV_MAXNREG;
    static constexpr bool CSR = true;
    static constexpr bool PDL_LATE = (CGVK_HS_LATE & 2) != 0;
    int mode;
    const double* pold;
    double* pnew;
    double alpha, beta;
    __device__ bool enter(const Params& P) {
        const Ctrl* c = P.ctrl;
        mode = c->mode2;
        if (mode == MODE_SKIP) return false;
        const int pc = c->pcur;
        pold = pc ? P.p1 : P.p0;
        pnew = pc ? P.p0 : P.p1;
        alpha = c->sc[SA];
        beta = c->sc[SB];
        return true;
    }
    __device__ const double* vec(const Params& P, int v) const {
        return v == 0 ? pold : v == 1 ? (PREC ? P.rt : P.r) : P.x;
    }
    static constexpr int NG = 2;  // gathered: p_old, r~ (combined as p = r~ + beta p_old)
    __device__ const double* gsrc(const Params& P, int k) const { return k == 0 ? pold : (PREC ? P.rt : P.r); }
    // band engine: its window holds p itself, formed once per column from the
    // two sources with the same expression as the on-the-fly gather
    static constexpr bool BAND_XF = true;
    __device__ double band_xf(double po, double rt) const { return ADD(rt, MUL(beta, po)); }
    __device__ int sync() const { return mode == MODE_FULL ? 2 : 1; }
    __device__ unsigned int* counter(const Params& P) const { return &P.ctrl->count[1]; }
    // split form (see cgvk_stream.cuh PairOf): the SpMV product, then the rest
    static constexpr bool PAIR = true;
    __device__ bool wants_spmv() const { return mode == MODE_FULL; }
    template <class In>
    __device__ auto gfun(const Params& P, const In& in) const {
        const double* __restrict__ rtv = PREC ? P.rt : P.r;
        const double* __restrict__ pg = pold;
        const double b = beta;
        return [=](int j) { return in.gather_p(j, rtv, pg, b); };
    }
    template <class In>
    __device__ void apply(const Params& P, int i, const In& in, double sum, double* acc) const {
        const double po = SV(0);
        st_far(P, P.x + i, ADD(SV(2), MUL(alpha, po)));
        if (mode != MODE_FULL) return;
        const double pi = ADD(SV(1), MUL(beta, po));
        pnew[i] = pi;
        P.s[i] = sum;
        acc[0] = ADD(acc[0], MUL(pi, sum));
    }
    template <class In, class RR>
    __device__ void row(const Params& P, int i, const In& in, const RR& R, double* acc) const {
        const double sum = wants_spmv() ? row_dot(R, gfun(P, in)) : 0.0;
        apply(P, i, in, sum, acc);
    }
    __device__ void finish(const Params& P, Ctrl* c, const double* tot) const {
        c->mode2 = MODE_SKIP;
        if (mode != MODE_FULL) return;
        c->pcur ^= 1;
        c->stats[STAT_SPMV] += 1;
        c->stats[STAT_RED] += 1;
        c->sc[SMU] = tot[0];
        if (settle_mu(c)) return;
        if (finalize_alpha(c)) return;
        check_tolerance(c);
    }
};

// ==================================================================  CG-CG
// src/variants.cpp:207-234. K1 = tail of step k-1 (p, s recurrences) + head
// of step k (x, r); K2 = w = A M r with nu, eta (+ unsimplified dots).

// streams: p s x r w [d]
template <bool PREC>
struct CgK1 {
    static constexpr int NV = PREC ? 6 : 5, ND = 0;
    static constexpr bool PDL_LATE = (CGVK_CG_LATE & 1) != 0;  // measured with G = 3 x SMs
    // no dots: sweeps downwards (cgvk_stream.cuh RevOf); measured CG V256 581 -> 574 us
    // (GV / pipe-PR's K2 reversed: V256 +6 / +27 us, left forward)
    static constexpr bool REVERSE = true;
    static constexpr bool CSR = false;
    bool F, S;
    double alpha, beta;
    __device__ bool enter(const Params& P) {
        const Ctrl* c = P.ctrl;
        F = c->form_pending != 0;
        S = step_wanted(c);
        alpha = c->sc[SA];
        beta = c->sc[SB];
        return F || S;
    }
    __device__ const double* vec(const Params& P, int v) const {
        switch (v) {
            case 0: return P.p0;
            case 1: return P.s;
            case 2: return S ? P.x : nullptr;
            case 3: return P.r;
            case 4: return F ? P.w : nullptr;
            default: return P.d;
        }
    }
    // steady state (F and S): every stream
    __device__ static const double* early_vec(const Params& P, int v) {
        const double* const e[6] = {P.p0, P.s, P.x, P.r, P.w, P.d};
        return e[v];
    }
    __device__ int sync() const { return (F && !S) ? 1 : 0; }
    __device__ unsigned int* counter(const Params& P) const { return &P.ctrl->count[0]; }
    template <class In, class RR>
    __device__ void row(const Params& P, int i, const In& in, const RR&, double*) const {
        double p = SV(0), s = SV(1);
        const double r = SV(3);
        if (F) {
            p = ADD(PREC ? MUL(SV(5), r) : r, MUL(beta, p));
            s = ADD(SV(4), MUL(beta, s));
            if (P.unsimplified_mu) {  // K2 reads them
                P.p0[i] = p;
                P.s[i] = s;
            } else {
                st_far(P, P.p0 + i, p);
                st_far(P, P.s + i, s);
            }
        }
        if (S) {
            st_far(P, P.x + i, ADD(SV(2), MUL(alpha, p)));
            const double rn = SUB(r, MUL(alpha, s));
            P.r[i] = rn;
            if constexpr (PREC) P.rt[i] = MUL(SV(5), rn);  // r~ = M r for K2's gather
        }
    }
    __device__ void finish(const Params&, Ctrl* c, const double*) const { c->form_pending = 0; }
};

// streams: A, r [d] [s p (unsimplified)]
template <bool PREC>
struct CgK2 {
    static constexpr int NV = 4, ND = 5;
    static constexpr bool PDL_LATE = (CGVK_CG_LATE & 2) != 0;
    static constexpr int MAXNREG = CGVK_SPMV_MAXNREG;
    static constexpr bool CSR = true;
    static constexpr int STAGES = 2;  // measured: a shallower ring leaves L1 to the gathers
    bool unsimp;
    __device__ bool enter(const Params& P) {
        unsimp = P.unsimplified_mu != 0;
        return step_wanted(P.ctrl);
    }
    __device__ const double* vec(const Params& P, int v) const { return early_vec(P, v); }
    __device__ static const double* early_vec(const Params& P, int v) {
        const bool u = P.unsimplified_mu != 0;
        switch (v) {
            case 0: return P.r;
            case 1: return PREC ? P.rt : nullptr;
            case 2: return u ? P.s : nullptr;
            default: return u ? P.p0 : nullptr;
        }
    }
    static constexpr int NG = 1;  // gathered: r~
    __device__ const double* gsrc(const Params& P, int) const { return PREC ? P.rt : P.r; }
    // dots: <r~,r> <r~,w> <r,r> [+ two with unsimplified_mu]
    __device__ static unsigned int dmask(const Params& P) { return P.unsimplified_mu ? 0x1fu : 0x07u; }
    __device__ int sync() const { return 2; }
    __device__ unsigned int* counter(const Params& P) const { return &P.ctrl->count[1]; }
    static constexpr bool PAIR = true;
    __device__ bool wants_spmv() const { return true; }
    template <class In>
    __device__ auto gfun(const Params& P, const In& in) const {
        const double* __restrict__ rtv = PREC ? P.rt : P.r;
        return [=](int j) { return in.gather(0, j, rtv); };
    }
    template <class In, class RR>
    __device__ void row(const Params& P, int i, const In& in, const RR& R, double* acc) const {
        apply(P, i, in, row_dot(R, gfun(P, in)), acc);
    }
    template <class In>
    __device__ void apply(const Params& P, int i, const In& in, double w, double* acc) const {
        P.w[i] = w;
        const double ri = SV(0), rti = PREC ? SV(1) : ri;
        acc[0] = ADD(acc[0], MUL(rti, ri));
        acc[1] = ADD(acc[1], MUL(rti, w));
        acc[2] = ADD(acc[2], MUL(ri, ri));
        if (unsimp) {
            acc[3] = ADD(acc[3], MUL(rti, SV(2)));  // <r~_k, s_{k-1}>
            acc[4] = ADD(acc[4], MUL(SV(3), w));    // <p_{k-1}, w_k>
        }
    }
    __device__ void finish(const Params& P, Ctrl* c, const double* tot) const {
        c->k += 1;
        c->stats[STAT_SPMV] += 1;
        c->stats[STAT_PREC] += PREC;
        c->stats[STAT_RED] += 2;
        record_rr(P, c, tot[2]);
        const double nu_next = tot[0];
        c->sc[SETA] = tot[1];
        c->form_pending = 0;
        if (settle_nonpositive(c, nu_next, BR_NU, tot[2])) {
            c->sc[SNU] = nu_next;
            return;
        }
        const double beta = DIV(nu_next, c->sc[SNU]);
        c->sc[SB] = beta;
        if (unsimp) c->stats[STAT_RED] += 2;
        const double mu_prev = c->sc[SMU];
        c->sc[SNU] = nu_next;
        c->form_pending = 1;  // p_k = M r_k + beta p, s_k = w_k + beta s (next K1)
        c->sc[SMU] = unsimp ? ADD(ADD(tot[1], MUL(beta, ADD(tot[3], tot[4]))), MUL(MUL(beta, beta), mu_prev))
                            : SUB(tot[1], MUL(DIV(beta, c->sc[SA]), nu_next));
        if (settle_mu(c)) return;
        if (finalize_alpha(c)) return;
        check_tolerance(c);
    }
};

// --------------------------------------------------- CG-CG, one kernel
// The same step (src/variants.cpp:207-234) as ONE launch per iteration for
// problems that fit L2 (see PrF below for the why). CG-CG has one global
// reduction per iteration; the K1 -> K2 boundary only carries r~ to the rows
// that gather it, and r~_j = d_j (r_j - alpha s_j) with s_j = w_j + beta s_j
// (when the beta-recurrences of the previous step are owed) is re-formed at
// every gathered column from the previous iteration's r, s, w with CgK1's
// expressions, operand order and rounding. r, s and w are double-buffered (a
// launch reads the set chosen by ctrl->pcur and writes the other; second
// buffers: P.u = r, P.t = s, P.p1 = w); p and x are updated in place; r~ is
// never stored (vector reads form d∘r). A form-only launch (materialize:
// F && !S) copies r and w forward, so the state stays in one set.
// streams: A, p s x r w [d]
template <bool PREC>
struct CgF {
    static constexpr int NV = PREC ? 6 : 5, ND = 5;
    static constexpr int MAXNREG = CGVK_SPMV_MAXNREG;
    static constexpr bool CSR = true;
    static constexpr bool PDL_LATE = (CGVK_F_LATE & 1) != 0;
    static constexpr bool NO_BAND = true;
    static constexpr bool NO_PEER = true;
    static constexpr int STAGES = 2;
    bool F, S, unsimp;
    double alpha, beta;
    const double *rc, *sc, *wc;  // this launch's inputs
    double *rn, *sn, *wn;        // its outputs
    __device__ bool enter(const Params& P) {
        const Ctrl* c = P.ctrl;
        F = c->form_pending != 0;
        S = step_wanted(c);
        unsimp = P.unsimplified_mu != 0;
        alpha = c->sc[SA];
        beta = c->sc[SB];
        const bool b = c->pcur != 0;
        rc = b ? P.u : P.r;
        rn = b ? P.r : P.u;
        sc = b ? P.t : P.s;
        sn = b ? P.s : P.t;
        wc = b ? P.p1 : P.w;
        wn = b ? P.w : P.p1;
        return F || S;
    }
    // whether a launch entered (and so flipped the buffer set), from the
    // control block it read (cgvk_stream.cuh HasEarlyPcur)
    __device__ static bool entered(const Ctrl* c) {
        return __ldcg(&c->form_pending) != 0 ||
               (__ldcg(&c->state) == ST_RUNNING && __ldcg(&c->k) < __ldcg(&c->k_limit));
    }
    __device__ const double* vec(const Params& P, int v) const { return early_vec(P, v, rc == P.u); }
    __device__ static const double* early_vec(const Params& P, int v, bool b) {
        switch (v) {
            case 0: return P.p0;
            case 1: return b ? P.t : P.s;
            case 2: return P.x;
            case 3: return b ? P.u : P.r;
            case 4: return b ? P.p1 : P.w;
            default: return P.d;
        }
    }
    static constexpr int NG = PREC ? 4 : 3;
    __device__ const double* gsrc(const Params& P, int k) const { return k == 0 ? rc : k == 1 ? sc : k == 2 ? wc : P.d; }
    // dots: <r~,r> <r~,w> <r,r> [+ two with unsimplified_mu]
    __device__ static unsigned int dmask(const Params& P) { return P.unsimplified_mu ? 0x1fu : 0x07u; }
    __device__ int sync() const { return S ? 2 : 1; }
    __device__ unsigned int* counter(const Params& P) const { return &P.ctrl->count[1]; }
    template <class In, class RR>
    __device__ void row(const Params& P, int i, const In& in, const RR& R, double* acc) const {
        // CgK1's row
        double p = SV(0), s = SV(1);
        const double r = SV(3);
        if (F) {
            p = ADD(PREC ? MUL(SV(5), r) : r, MUL(beta, p));
            s = ADD(SV(4), MUL(beta, s));
            P.p0[i] = p;
        }
        sn[i] = s;
        if (!S) {  // form only: r, w unchanged
            rn[i] = r;
            wn[i] = SV(4);
            return;
        }
        P.x[i] = ADD(SV(2), MUL(alpha, p));
        const double ri = SUB(r, MUL(alpha, s));
        rn[i] = ri;
        const double rti = PREC ? MUL(SV(5), ri) : ri;
        // CgK2's row, r~ re-formed at every gathered column
        const double* __restrict__ rg = rc;
        const double* __restrict__ sg = sc;
        const double* __restrict__ wg = wc;
        const double* __restrict__ dg = P.d;
        const double a = alpha, b = beta;
        const bool f = F;
        const double w = row_dot(R, [=](int j) {
            // (branch-free: w_j is loaded even when no recurrence is owed, so
            // a chunk's loads all issue before its arithmetic)
            const double s0 = in.gather(1, j, sg);
            const double sf = ADD(in.gather(2, j, wg), MUL(b, s0));
            const double sj = f ? sf : s0;
            const double rj = SUB(in.gather(0, j, rg), MUL(a, sj));
            return PREC ? MUL(in.gather(3, j, dg), rj) : rj;
        });
        wn[i] = w;
        acc[0] = ADD(acc[0], MUL(rti, ri));
        acc[1] = ADD(acc[1], MUL(rti, w));
        acc[2] = ADD(acc[2], MUL(ri, ri));
        if (unsimp) {
            acc[3] = ADD(acc[3], MUL(rti, s));  // <r~_k, s_{k-1}>
            acc[4] = ADD(acc[4], MUL(p, w));    // <p_{k-1}, w_k>
        }
    }
    __device__ void finish(const Params& P, Ctrl* c, const double* tot) const {
        c->pcur ^= 1;
        if (!S) {
            c->form_pending = 0;
            return;
        }
        CgK2<PREC> k2;
        k2.unsimp = unsimp;
        k2.finish(P, c, tot);
    }
};

// ===============================================================  PR / M
// src/variants.cpp:237-265, paper Alg. 2 (M-CG with the Meurant nu').
// K1: x, r, r~ (s~ = M s on the fly) and p; K2: s = A p with mu, delta,
// delta-hat, gamma (s~ on the fly), nu, <r,r>.

// streams: x p r s [r~ d]
template <bool PREC>
#ifndef CGVK_PR_K1_CTAS
#define CGVK_PR_K1_CTAS 3
#endif
#ifndef CGVK_PR_LATE
#define CGVK_PR_LATE 2  // bit 0: K1, bit 1: K2 signal their dependents late
#endif
struct PrK1 {
    static constexpr int NV = PREC ? 6 : 4, ND = 1;
    static constexpr bool CSR = false;
    // measured P128: 3 resident CTAs + late PDL signal, PR 70.5 -> 67.9 us;
    // with the chained schedule an early signal is as fast at P128 and 5 % faster at P64
    static constexpr int SMEM_CTAS = CGVK_PR_K1_CTAS;
    static constexpr bool PDL_LATE = (CGVK_PR_LATE & 1) != 0;
    double alpha, beta, nup;
    bool valid;
    __device__ bool enter(const Params& P) {
        const Ctrl* c = P.ctrl;
        if (!step_wanted(c)) return false;
        alpha = c->sc[SA];
        nup = predicted_nu(P.nu_expr, c->sc);
        valid = isfinite(nup) && nup > 0.0;
        beta = DIV(nup, c->sc[SNU]);
        return true;
    }
    __device__ const double* vec(const Params& P, int v) const { return early_vec(P, v); }
    __device__ static const double* early_vec(const Params& P, int v) {
        switch (v) {
            case 0: return P.x;
            case 1: return P.p0;
            case 2: return P.r;
            case 3: return P.s;
            case 4: return P.rt;
            default: return P.d;
        }
    }
    __device__ int sync() const { return valid ? 0 : 2; }
    __device__ unsigned int* counter(const Params& P) const { return &P.ctrl->count[0]; }
    template <class In, class RR>
    __device__ void row(const Params& P, int i, const In& in, const RR&, double* acc) const {
        const double s = SV(3), p = SV(1);
        st_far(P, P.x + i, ADD(SV(0), MUL(alpha, p)));
        const double r = SUB(SV(2), MUL(alpha, s));
        P.r[i] = r;
        double rt = r;
        if constexpr (PREC) {
            rt = SUB(SV(4), MUL(alpha, MUL(SV(5), s)));
            P.rt[i] = rt;
        }
        if (valid)
            P.p0[i] = ADD(rt, MUL(beta, p));
        else
            acc[0] = ADD(acc[0], MUL(r, r));
    }
    __device__ void finish(const Params& P, Ctrl* c, const double* tot) const {
        c->k += 1;
        c->sc[SNUP] = nup;
        record_rr(P, c, tot[0]);
        settle_nonpositive(c, nup, BR_NUPRIME, tot[0]);
    }
};

// streams: A, p r [r~ d]
template <bool PREC>
struct PrK2 {
    static constexpr int NV = PREC ? 4 : 2, ND = 6;
    static constexpr int MAXNREG = CGVK_SPMV_MAXNREG;
    static constexpr bool CSR = true;
    static constexpr bool PDL_LATE = (CGVK_PR_LATE & 2) != 0;
    double nup;
    bool want_delta, want_dhat;
    __device__ bool enter(const Params& P) {
        const Ctrl* c = P.ctrl;
        if (!step_wanted(c)) return false;
        nup = predicted_nu(P.nu_expr, c->sc);
        want_delta = P.nu_expr != 2 || P.track_delta;
        want_dhat = P.nu_expr == 0;
        return isfinite(nup) && nup > 0.0;
    }
    __device__ const double* vec(const Params& P, int v) const { return early_vec(P, v); }
    __device__ static const double* early_vec(const Params& P, int v) {
        return v == 0 ? P.p0 : v == 1 ? P.r : v == 2 ? P.rt : P.d;
    }
    static constexpr int NG = 1;  // gathered: p
    __device__ const double* gsrc(const Params& P, int) const { return P.p0; }
    __device__ int sync() const { return 2; }
    __device__ unsigned int* counter(const Params& P) const { return &P.ctrl->count[1]; }
    static constexpr bool PAIR = true;
    __device__ bool wants_spmv() const { return true; }
    template <class In>
    __device__ auto gfun(const Params& P, const In& in) const {
        const double* __restrict__ p = P.p0;
        return [=](int j) { return in.gather(0, j, p); };
    }
    template <class In, class RR>
    __device__ void row(const Params& P, int i, const In& in, const RR& R, double* acc) const {
        apply(P, i, in, row_dot(R, gfun(P, in)), acc);
    }
    template <class In>
    __device__ void apply(const Params& P, int i, const In& in, double s, double* acc) const {
        P.s[i] = s;
        const double st = PREC ? MUL(SV(3), s) : s;
        const double r = SV(1);
        const double rt = PREC ? SV(2) : r;
        acc[0] = ADD(acc[0], MUL(SV(0), s));
        if (want_delta) acc[1] = ADD(acc[1], MUL(rt, s));
        if (want_dhat) acc[2] = ADD(acc[2], MUL(st, r));
        acc[3] = ADD(acc[3], MUL(st, s));
        acc[4] = ADD(acc[4], MUL(rt, r));
        acc[5] = ADD(acc[5], MUL(r, r));
    }
    __device__ void finish(const Params& P, Ctrl* c, const double* tot) const {
        c->k += 1;
        c->sc[SNUP] = nup;
        c->sc[SB] = DIV(nup, c->sc[SNU]);
        c->stats[STAT_SPMV] += 1;
        c->stats[STAT_PREC] += PREC;
        c->stats[STAT_RED] += 2 + want_delta + want_dhat;
        record_rr(P, c, tot[5]);
        c->sc[SMU] = tot[0];
        if (want_delta) c->sc[SDEL] = tot[1];
        if (want_dhat) c->sc[SDELH] = tot[2];
        c->sc[SGAM] = tot[3];
        if (settle_mu(c)) return;
        if (P.recompute_nu) {
            c->stats[STAT_RED] += 1;
            const double nu_next = tot[4];
            if (settle_nonpositive(c, nu_next, BR_NU, tot[5])) {
                c->sc[SNU] = nu_next;
                return;
            }
            c->sc[SNU] = nu_next;
        } else {
            c->sc[SNU] = nup;
        }
        if (finalize_alpha(c)) return;
        check_tolerance(c);
    }
};

// ---------------------------------------------------- PR / M, one kernel
// The same step (src/variants.cpp:237-265) as ONE launch per iteration, for
// problems whose working set fits L2 (launch- and latency-bound: each kernel
// boundary costs 3-5 us of drain, dependency release, scalar prologue and
// pipeline fill against a ~3 us tile pass). PR has one global reduction per
// iteration, so one boundary is all it needs: the K1 -> K2 boundary only
// carries p to the rows that gather it, and p_j = r~_j + beta p_j with
// r~_j = r~_j - alpha (d_j s_j) is re-formed at every gathered column from the
// previous iteration's r~, s, p (the expression, operand order and rounding
// of PrK1::row, so the same bits) — as HsK2 forms its p on the fly. The
// vectors other rows gather (p, s and r~, or r without a preconditioner) are
// double-buffered: a launch reads the set chosen by ctrl->pcur and writes the
// other one (second buffers: P.p1, P.w = s, P.u = r~ | r); x (and r with
// Jacobi) are updated in place. A breakdown of nu' (PrK1's `valid == false`)
// copies p and s forward unchanged, so the state stays in one buffer set.
// Dots, their canonical order and the scalar tail are PrK2's (PrK1's on that
// breakdown). The launch chains with itself (chain_prologue<PrF, PrF>).
// streams: A, x p r s [r~ d]
template <bool PREC>
struct PrF {
    static constexpr int NV = PREC ? 6 : 4, ND = 6;
    static constexpr int MAXNREG = CGVK_SPMV_MAXNREG;
    static constexpr bool CSR = true;
    static constexpr bool PDL_LATE = CGVK_PRF_LATE != 0;
    static constexpr bool NO_BAND = true;
    double alpha, beta, nup;
    bool valid, want_delta, want_dhat;
    const double *pc, *sc, *gc;  // this iteration's inputs: p, s and g = r~ (Jacobi) | r
    double *pn, *sn, *gn;        // its outputs
    __device__ bool enter(const Params& P) {
        const Ctrl* c = P.ctrl;
        if (!step_wanted(c)) return false;
        alpha = c->sc[SA];
        nup = predicted_nu(P.nu_expr, c->sc);
        valid = isfinite(nup) && nup > 0.0;
        beta = DIV(nup, c->sc[SNU]);
        want_delta = P.nu_expr != 2 || P.track_delta;
        want_dhat = P.nu_expr == 0;
        double* const g0 = PREC ? P.rt : P.r;
        const bool b = c->pcur != 0;
        pc = b ? P.p1 : P.p0;
        pn = b ? P.p0 : P.p1;
        sc = b ? P.w : P.s;
        sn = b ? P.s : P.w;
        gc = b ? P.u : g0;
        gn = b ? g0 : P.u;
        return true;
    }
    __device__ static bool entered(const Ctrl* c) {  // (cgvk_stream.cuh HasEarlyPcur)
        return __ldcg(&c->state) == ST_RUNNING && __ldcg(&c->k) < __ldcg(&c->k_limit);
    }
    __device__ const double* vec(const Params& P, int v) const { return CGVK_PRF_EVEC(P, v, pc == P.p1); }
    // the streams given the buffer-set bit (cgvk_stream.cuh HasEarlyPcur)
    __device__ static const double* CGVK_PRF_EVEC(const Params& P, int v, bool b) {
        const double* const g = b ? P.u : (PREC ? P.rt : P.r);
        switch (v) {
            case 0: return P.x;
            case 1: return b ? P.p1 : P.p0;
            case 2: return PREC ? P.r : g;
            case 3: return b ? P.w : P.s;
            case 4: return g;
            default: return P.d;
        }
    }
    static constexpr int NG = PREC ? 4 : 3;
    __device__ const double* gsrc(const Params& P, int k) const { return k == 0 ? pc : k == 1 ? sc : k == 2 ? gc : P.d; }
    __device__ int sync() const { return 2; }
    __device__ unsigned int* counter(const Params& P) const { return &P.ctrl->count[1]; }
    template <class In, class RR>
    __device__ void row(const Params& P, int i, const In& in, const RR& R, double* acc) const {
        // PrK1's row
        const double s = SV(3), p = SV(1);
        P.x[i] = ADD(SV(0), MUL(alpha, p));
        const double r = SUB(SV(2), MUL(alpha, s));
        double rt = r;
        if constexpr (PREC) {
            P.r[i] = r;
            rt = SUB(SV(4), MUL(alpha, MUL(SV(5), s)));
        }
        gn[i] = rt;
        if (!valid) {  // its breakdown step: p, s unchanged, <r,r> for the record
            pn[i] = p;
            sn[i] = s;
            acc[5] = ADD(acc[5], MUL(r, r));
            return;
        }
        const double pi = ADD(rt, MUL(beta, p));
        pn[i] = pi;
        // PrK2's row, p re-formed at every gathered column
        const double* __restrict__ pg = pc;
        const double* __restrict__ sg = sc;
        const double* __restrict__ gg = gc;
        const double* __restrict__ dg = P.d;
        const double a = alpha, b = beta;
        const double sum = row_dot(R, [=](int j) {
            const double sj = in.gather(1, j, sg);
            const double gj = in.gather(2, j, gg);
            const double rtj = SUB(gj, MUL(a, PREC ? MUL(in.gather(3, j, dg), sj) : sj));
            return ADD(rtj, MUL(b, in.gather(0, j, pg)));
        });
        sn[i] = sum;
        const double st = PREC ? MUL(SV(5), sum) : sum;
        acc[0] = ADD(acc[0], MUL(pi, sum));
        if (want_delta) acc[1] = ADD(acc[1], MUL(rt, sum));
        if (want_dhat) acc[2] = ADD(acc[2], MUL(st, r));
        acc[3] = ADD(acc[3], MUL(st, sum));
        acc[4] = ADD(acc[4], MUL(rt, r));
        acc[5] = ADD(acc[5], MUL(r, r));
    }
    __device__ void finish(const Params& P, Ctrl* c, const double* tot) const {
        c->pcur ^= 1;
        if (!valid) {
            PrK1<PREC> k1;
            k1.nup = nup;
            const double t0[1] = {tot[5]};
            k1.finish(P, c, t0);
            return;
        }
        PrK2<PREC> k2;
        k2.nup = nup;
        k2.want_delta = want_delta;
        k2.want_dhat = want_dhat;
        k2.finish(P, c, tot);
    }
};

// ====================================================================  GV
// src/variants.cpp:267-298. K1 = beta-recurrences of step k-1 (p, s, s~, u)
// + step k updates (x, r, r~, w) with nu, eta; the reduction is folded at the
// end of K1, so on multi-GPU it overlaps K2 = t = A M w.

// streams: p s u w t x r [s~ r~ d]
template <bool PREC>
struct GvK1 {
    static constexpr int NV = PREC ? 10 : 7, ND = 5;
    static constexpr bool PDL_LATE = (CGVK_GV_LATE & 1) != 0;  // measured with G = 3 x SMs
    static constexpr int MAXNREG = CGVK_K1_MAXNREG;
    static constexpr int SMEM_CTAS = CGVK_GV_K1_CTAS;
    static constexpr bool CSR = false;
    bool F, S, unsimp;
    double alpha, beta;
    __device__ bool enter(const Params& P) {
        const Ctrl* c = P.ctrl;
        F = c->form_pending != 0;
        S = step_wanted(c);
        alpha = c->sc[SA];
        beta = c->sc[SB];
        unsimp = P.unsimplified_mu != 0;
        return F || S;
    }
    __device__ const double* vec(const Params& P, int v) const {
        switch (v) {
            case 0: return P.p0;
            case 1: return P.s;
            case 2: return P.u;
            case 3: return P.w;
            case 4: return F ? P.t : nullptr;
            case 5: return S ? P.x : nullptr;
            case 6: return P.r;
            case 7: return P.st;
            case 8: return P.rt;
            default: return P.d;
        }
    }
    // (no early_vec: measured P64 GV 18.9 -> 20.9 us with it — ten streams
    // per stage issued at once delay the chained prologue; with the successor
    // fold 15.6 -> 16.3 us)
    // dots: <r~,r> <r~,w> <r,r> [+ two with unsimplified_mu]
    __device__ static unsigned int dmask(const Params& P) { return P.unsimplified_mu ? 0x1fu : 0x07u; }
    __device__ int sync() const { return S ? 2 : 1; }
    __device__ unsigned int* counter(const Params& P) const { return &P.ctrl->count[0]; }
    template <class In, class RR>
    __device__ void row(const Params& P, int i, const In& in, const RR&, double* acc) const {
        double p = SV(0), s = SV(1), u = SV(2), w = SV(3);
        double st = PREC ? SV(7) : s;
        double rt = PREC ? SV(8) : SV(6);
        if (F) {
            p = ADD(rt, MUL(beta, p));
            s = ADD(w, MUL(beta, s));
            if constexpr (PREC) st = ADD(MUL(SV(9), w), MUL(beta, st));
            else st = s;
            u = ADD(SV(4), MUL(beta, u));
            st_far(P, P.p0 + i, p);
            st_far(P, P.s + i, s);
            if constexpr (PREC) st_far(P, P.st + i, st);
            st_far(P, P.u + i, u);
        }
        if (S) {
            st_far(P, P.x + i, ADD(SV(5), MUL(alpha, p)));
            const double r = SUB(SV(6), MUL(alpha, s));
            st_far(P, P.r + i, r);
            if constexpr (PREC) {
                rt = SUB(rt, MUL(alpha, st));
                st_far(P, P.rt + i, rt);
            } else {
                rt = r;
            }
            w = SUB(w, MUL(alpha, u));
            if constexpr (PREC) {
                st_far(P, P.w + i, w);
                P.wt[i] = MUL(SV(9), w);  // w~ = M w for K2's gather
            } else {
                P.w[i] = w;
            }
            acc[0] = ADD(acc[0], MUL(rt, r));
            acc[1] = ADD(acc[1], MUL(rt, w));
            acc[2] = ADD(acc[2], MUL(r, r));
            if (unsimp) {
                acc[3] = ADD(acc[3], MUL(rt, s));  // <r~_k, s_{k-1}>
                acc[4] = ADD(acc[4], MUL(p, w));   // <p_{k-1}, w_k>
            }
        }
    }
    // row-partitioned: K2 (t = A w~) may start before the exchanged reduction
    // is finalised, so its go-ahead is set here, by K1 itself
    __device__ void dist_mark(const Params&, Ctrl* c) const {
        if (S) c->mode2 = MODE_FULL;
    }
    __device__ void finish(const Params& P, Ctrl* c, const double* tot) const {
        if (!S) {  // materialisation only
            c->form_pending = 0;
            return;
        }
        c->k += 1;
        if (!P.dist) c->mode2 = MODE_FULL;  // t = A w~ precedes the checks in the reference
        c->stats[STAT_SPMV] += 1;
        c->stats[STAT_PREC] += PREC;
        c->stats[STAT_RED] += 2;
        record_rr(P, c, tot[2]);
        const double nu_next = tot[0];
        c->sc[SETA] = tot[1];
        c->form_pending = 0;
        if (settle_nonpositive(c, nu_next, BR_NU, tot[2])) {
            c->sc[SNU] = nu_next;
            return;
        }
        const double beta_k = DIV(nu_next, c->sc[SNU]);
        c->sc[SB] = beta_k;
        if (unsimp) c->stats[STAT_RED] += 2;
        const double mu_prev = c->sc[SMU];
        c->sc[SNU] = nu_next;
        c->form_pending = 1;
        c->sc[SMU] = unsimp ? ADD(ADD(tot[1], MUL(beta_k, ADD(tot[3], tot[4]))), MUL(MUL(beta_k, beta_k), mu_prev))
                            : SUB(tot[1], MUL(DIV(beta_k, c->sc[SA]), nu_next));
        if (settle_mu(c)) return;
        if (finalize_alpha(c)) return;
        check_tolerance(c);
    }
};

// t = A M w (streams: A; gathers w~ = M w stored by K1)
template <bool PREC>
struct GvK2 {
    static constexpr int NV = 0, ND = 0;
    static constexpr bool PDL_LATE = (CGVK_GV_LATE & 2) != 0;
    static constexpr int MAXNREG = CGVK_SPMV_MAXNREG;
    static constexpr bool CSR = true;
    // measured: 2 stages at 4 CTAs/SM (G = 12 x SMs); with G = 3 x SMs the grid
    // is 3 CTAs/SM and a 3-stage ring is faster (V256 GV 740 -> 697 us)
    static constexpr int STAGES = 3;
    __device__ bool enter(const Params& P) { return P.ctrl->mode2 != MODE_SKIP; }
    __device__ const double* vec(const Params&, int) const { return nullptr; }
    static constexpr int NG = 1;  // gathered: w~
    __device__ const double* gsrc(const Params& P, int) const { return PREC ? P.wt : P.w; }
    __device__ int sync() const { return 1; }
    __device__ unsigned int* counter(const Params& P) const { return &P.ctrl->count[1]; }
    static constexpr bool PAIR = true;
    __device__ bool wants_spmv() const { return true; }
    template <class In>
    __device__ auto gfun(const Params& P, const In& in) const {
        const double* __restrict__ wtv = PREC ? P.wt : P.w;  // w~ stored by K1
        return [=](int j) { return in.gather(0, j, wtv); };
    }
    template <class In>
    __device__ void apply(const Params& P, int i, const In&, double t, double*) const { P.t[i] = t; }
    template <class In, class RR>
    __device__ void row(const Params& P, int i, const In& in, const RR& R, double* acc) const {
        apply(P, i, in, row_dot(R, gfun(P, in)), acc);
    }
    __device__ void finish(const Params&, Ctrl* c, const double*) const { c->mode2 = MODE_SKIP; }
};

// ------------------------------------------------------ GV, one kernel
// The same step (src/variants.cpp:267-298) as ONE launch per iteration for a
// single-GPU problem that fits L2 (see PrF above for the why; a row-
// partitioned solve keeps two kernels — there K1's reduction overlaps K2).
// The K1 -> K2 boundary only carries w~ to the rows that gather it, and
// w~_j = d_j (w_j - alpha u_j) with u_j = t_j + beta u_j (when the
// beta-recurrences are owed) is re-formed at every gathered column from the
// previous iteration's w, u, t with GvK1's expressions and rounding. w, u and
// t are double-buffered (second buffers P.b0 / b1 / b2, set chosen by
// ctrl->pcur); everything else is updated in place; w~ is never stored. The
// SpMV runs before the step's checks are known, as in the reference.
// streams: A, p s u w t x r [s~ r~ d]
template <bool PREC>
struct GvF {
    static constexpr int NV = PREC ? 10 : 7, ND = 5;
    static constexpr int MAXNREG = CGVK_SPMV_MAXNREG;
    static constexpr bool CSR = true;
    static constexpr bool PDL_LATE = (CGVK_F_LATE & 2) != 0;
    static constexpr bool NO_BAND = true;
    static constexpr bool NO_PEER = true;
    static constexpr int STAGES = 2;
    static constexpr int MINB = 2;       // GvK1's register appetite
    static constexpr int SMEM_CTAS = 2;
    bool F, S, unsimp;
    double alpha, beta;
    const double *wc, *uc, *tc;
    double *wn, *un, *tn;
    __device__ bool enter(const Params& P) {
        const Ctrl* c = P.ctrl;
        F = c->form_pending != 0;
        S = step_wanted(c);
        alpha = c->sc[SA];
        beta = c->sc[SB];
        unsimp = P.unsimplified_mu != 0;
        const bool b = c->pcur != 0;
        wc = b ? P.b0 : P.w;
        wn = b ? P.w : P.b0;
        uc = b ? P.b1 : P.u;
        un = b ? P.u : P.b1;
        tc = b ? P.b2 : P.t;
        tn = b ? P.t : P.b2;
        return F || S;
    }
    __device__ static bool entered(const Ctrl* c) { return CgF<PREC>::entered(c); }
    __device__ const double* vec(const Params& P, int v) const { return early_vec(P, v, wc == P.b0); }
    __device__ static const double* early_vec(const Params& P, int v, bool b) {
        switch (v) {
            case 0: return P.p0;
            case 1: return P.s;
            case 2: return b ? P.b1 : P.u;
            case 3: return b ? P.b0 : P.w;
            case 4: return b ? P.b2 : P.t;
            case 5: return P.x;
            case 6: return P.r;
            case 7: return P.st;
            case 8: return P.rt;
            default: return P.d;
        }
    }
    static constexpr int NG = PREC ? 4 : 3;
    __device__ const double* gsrc(const Params& P, int k) const { return k == 0 ? wc : k == 1 ? uc : k == 2 ? tc : P.d; }
    // dots: <r~,r> <r~,w> <r,r> [+ two with unsimplified_mu]
    __device__ static unsigned int dmask(const Params& P) { return P.unsimplified_mu ? 0x1fu : 0x07u; }
    __device__ int sync() const { return S ? 2 : 1; }
    __device__ unsigned int* counter(const Params& P) const { return &P.ctrl->count[1]; }
    template <class In, class RR>
    __device__ void row(const Params& P, int i, const In& in, const RR& R, double* acc) const {
        // GvK1's row
        double p = SV(0), s = SV(1), u = SV(2), w = SV(3);
        double st = PREC ? SV(7) : s;
        double rt = PREC ? SV(8) : SV(6);
        if (F) {
            p = ADD(rt, MUL(beta, p));
            s = ADD(w, MUL(beta, s));
            if constexpr (PREC) st = ADD(MUL(SV(9), w), MUL(beta, st));
            else st = s;
            u = ADD(SV(4), MUL(beta, u));
            P.p0[i] = p;
            P.s[i] = s;
            if constexpr (PREC) P.st[i] = st;
        }
        un[i] = u;
        if (!S) {  // form only: w, t unchanged
            wn[i] = w;
            tn[i] = SV(4);
            return;
        }
        P.x[i] = ADD(SV(5), MUL(alpha, p));
        const double r = SUB(SV(6), MUL(alpha, s));
        P.r[i] = r;
        if constexpr (PREC) {
            rt = SUB(rt, MUL(alpha, st));
            P.rt[i] = rt;
        } else {
            rt = r;
        }
        w = SUB(w, MUL(alpha, u));
        wn[i] = w;
        acc[0] = ADD(acc[0], MUL(rt, r));
        acc[1] = ADD(acc[1], MUL(rt, w));
        acc[2] = ADD(acc[2], MUL(r, r));
        if (unsimp) {
            acc[3] = ADD(acc[3], MUL(rt, s));  // <r~_k, s_{k-1}>
            acc[4] = ADD(acc[4], MUL(p, w));   // <p_{k-1}, w_k>
        }
        // GvK2's row, w~ re-formed at every gathered column (branch-free)
        const double* __restrict__ wg = wc;
        const double* __restrict__ ug = uc;
        const double* __restrict__ tg = tc;
        const double* __restrict__ dg = P.d;
        const double a = alpha, b = beta;
        const bool f = F;
        tn[i] = row_dot(R, [=](int j) {
            const double u0 = in.gather(1, j, ug);
            const double uf = ADD(in.gather(2, j, tg), MUL(b, u0));
            const double uj = f ? uf : u0;
            const double wj = SUB(in.gather(0, j, wg), MUL(a, uj));
            return PREC ? MUL(in.gather(3, j, dg), wj) : wj;
        });
    }
    __device__ void finish(const Params& P, Ctrl* c, const double* tot) const {
        c->pcur ^= 1;
        GvK1<PREC> k1;
        k1.S = S;
        k1.unsimp = unsimp;
        k1.finish(P, c, tot);
        c->mode2 = MODE_SKIP;  // (GvK2's finish: the SpMV is done)
    }
};

// ===============================================================  pipe-PR
// src/variants.cpp:303-350, paper Alg. 3 and the §2.2.1 schedule
// (PAPER.md:384-401): every dot of step k is computed in K1 from the updated
// vectors (they do not depend on u, w), so its reduction overlaps the block
// SpMV K2 = (u, w) = A (s~, r~). w~ = M w and u~ = M u are recomputed on the
// fly (recompute_w); with recompute_w off, w and w~ are stored recurrences.

// streams: x p r s w u [s~ r~ d w~]
template <bool PREC>
struct PprK1 {
    static constexpr int NV = PREC ? 10 : 6, ND = 6;
    static constexpr bool PDL_LATE = (CGVK_PPR_LATE & 1) != 0;
    static constexpr int MAXNREG = CGVK_K1_MAXNREG;
    static constexpr int SMEM_CTAS = CGVK_PPR_K1_CTAS;
    static constexpr bool RR2 = true;  // two virtual CTAs per CTA interleaved (cgvk_stream.cuh rr2_tile)
    static constexpr bool CSR = false;
    double alpha, beta, nup;
    bool valid, want_delta, want_dhat, recw;
    __device__ bool enter(const Params& P) {
        const Ctrl* c = P.ctrl;
        if (!step_wanted(c)) return false;
        alpha = c->sc[SA];
        nup = predicted_nu(P.nu_expr, c->sc);
        valid = isfinite(nup) && nup > 0.0;
        beta = DIV(nup, c->sc[SNU]);
        want_delta = P.nu_expr != 2 || P.track_delta;
        want_dhat = P.nu_expr == 0;
        recw = P.recompute_w != 0;
        return true;
    }
    __device__ const double* vec(const Params& P, int v) const {
        switch (v) {
            case 0: return P.x;
            case 1: return P.p0;
            case 2: return P.r;
            case 3: return P.s;
            case 4: return P.w;
            case 5: return P.u;
            case 6: return P.st;
            case 7: return P.rt;
            case 8: return P.d;
            default: return recw ? nullptr : P.wt;
        }
    }
    // (no early_vec: measured P64 pipe-PR 21.1 -> 22.9 us with it; with the
    // successor fold 17.0 -> 17.4, P128 80.7 -> 85.5)
    __device__ int sync() const { return 2; }
    __device__ unsigned int* counter(const Params& P) const { return &P.ctrl->count[0]; }
    // row-partitioned: the block SpMV's go-ahead, set by K1 (see GvK1)
    __device__ void dist_mark(const Params&, Ctrl* c) const {
        if (valid) c->mode2 = MODE_FULL;
    }
    template <class In, class RR>
    __device__ void row(const Params& P, int i, const In& in, const RR&, double* acc) const {
        const double p_old = SV(1), s_old = SV(3), w_old = SV(4), u = SV(5);
        st_far(P, P.x + i, ADD(SV(0), MUL(alpha, p_old)));
        const double r = SUB(SV(2), MUL(alpha, s_old));
        if (PREC) st_far(P, P.r + i, r);  // (without Jacobi K2 gathers r)
        else P.r[i] = r;
        double rt = r, st_old = s_old;
        if constexpr (PREC) {
            st_old = SV(6);
            rt = SUB(SV(7), MUL(alpha, st_old));
            P.rt[i] = rt;
        }
        const double wn = SUB(w_old, MUL(alpha, u));  // w'_k
        if (P.wpred) P.wpred[i] = wn;                  // run()'s probes track the prediction
        double wtn = wn;
        if constexpr (PREC) {
            const double d = SV(8);
            const double wt_old = recw ? MUL(d, w_old) : SV(9);
            wtn = SUB(wt_old, MUL(alpha, MUL(d, u)));
        }
        if (valid) {
            const double p = ADD(rt, MUL(beta, p_old));
            const double s = ADD(wn, MUL(beta, s_old));
            double st = s;
            if constexpr (PREC) {
                st = ADD(wtn, MUL(beta, st_old));
                P.st[i] = st;
            }
            st_far(P, P.p0 + i, p);
            if (PREC) st_far(P, P.s + i, s);  // (without Jacobi K2 gathers s)
            else P.s[i] = s;
            if (!recw) {
                st_far(P, P.w + i, wn);
                if constexpr (PREC) st_far(P, P.wt + i, wtn);
            }
            acc[0] = ADD(acc[0], MUL(p, s));
            if (want_delta) acc[1] = ADD(acc[1], MUL(rt, s));
            if (want_dhat) acc[2] = ADD(acc[2], MUL(st, r));
            acc[3] = ADD(acc[3], MUL(st, s));
            acc[4] = ADD(acc[4], MUL(rt, r));
        } else {
            P.w[i] = wn;
            if constexpr (PREC) P.wt[i] = wtn;
        }
        acc[5] = ADD(acc[5], MUL(r, r));
    }
    __device__ void finish(const Params& P, Ctrl* c, const double* tot) const {
        c->k += 1;
        c->sc[SNUP] = nup;
        record_rr(P, c, tot[5]);
        if (!valid) {
            c->wt_stored = PREC;
            settle_nonpositive(c, nup, BR_NUPRIME, tot[5]);
            return;
        }
        c->sc[SB] = beta;
        if (!P.dist) c->mode2 = MODE_FULL;  // the block SpMV precedes the checks in the reference
        if (recw) {
            c->stats[STAT_BLOCK] += 1;
            c->stats[STAT_PREC] += 2 * PREC;
        } else {
            c->stats[STAT_SPMV] += 1;
            c->stats[STAT_PREC] += PREC;
        }
        c->stats[STAT_RED] += 2 + want_delta + want_dhat;
        c->sc[SMU] = tot[0];
        if (want_delta) c->sc[SDEL] = tot[1];
        if (want_dhat) c->sc[SDELH] = tot[2];
        c->sc[SGAM] = tot[3];
        if (settle_mu(c)) return;
        if (P.recompute_nu) {
            c->stats[STAT_RED] += 1;
            const double nu_next = tot[4];
            if (settle_nonpositive(c, nu_next, BR_NU, tot[5])) {
                c->sc[SNU] = nu_next;
                return;
            }
            c->sc[SNU] = nu_next;
        } else {
            c->sc[SNU] = nup;
        }
        if (finalize_alpha(c)) return;
        check_tolerance(c);
    }
};

// (u, w) = A (s~, r~) in one traversal, or u = A s~ with recompute_w off
// (streams: A; gathers s~, r~)
template <bool PREC>
struct PprK2 {
    static constexpr int NV = 0, ND = 0;
    static constexpr bool PDL_LATE = (CGVK_PPR_LATE & 2) != 0;
    static constexpr int MAXNREG = CGVK_SPMV_MAXNREG;
    static constexpr bool CSR = true;
    bool recw;
    __device__ bool enter(const Params& P) {
        recw = P.recompute_w != 0;
        return P.ctrl->mode2 != MODE_SKIP;
    }
    __device__ const double* vec(const Params&, int) const { return nullptr; }
    static constexpr int NG = 2;  // gathered: s~, r~ (the latter only with recompute_w)
    __device__ const double* gsrc(const Params& P, int k) const {
        if (k == 0) return PREC ? P.st : P.s;
        return recw ? (PREC ? P.rt : P.r) : nullptr;
    }
    __device__ int sync() const { return 1; }
    __device__ unsigned int* counter(const Params& P) const { return &P.ctrl->count[1]; }
    template <class In, class RR>
    __device__ void row(const Params& P, int i, const In& in, const RR& R, double*) const {
        const double* __restrict__ sv_ = PREC ? P.st : P.s;
        const double* __restrict__ rv = PREC ? P.rt : P.r;
        if (recw) {
            double u, w;
            row_dot2(R, [&](int j) { return in.gather(0, j, sv_); },
                     [&](int j) { return in.gather(1, j, rv); }, u, w);
            P.u[i] = u;
            P.w[i] = w;
        } else {
            P.u[i] = row_dot(R, [&](int j) { return in.gather(0, j, sv_); });
        }
    }
    __device__ void finish(const Params&, Ctrl* c, const double*) const { c->mode2 = MODE_SKIP; }
};

// -------------------------------------------------- pipe-PR, one kernel
// The same step (src/variants.cpp:303-350, recompute_w on) as ONE launch per
// iteration for a single-GPU problem with at most one tile per resident CTA
// (see PrF / GvF for the why; a row-partitioned solve keeps two kernels —
// there K1's reduction overlaps the block SpMV). The K1 -> K2 boundary only
// carries s~ and r~ to the rows that gather them; both are re-formed at every
// gathered column from the previous iteration's s~, r~, w, u (and Jacobi's d)
// with PprK1's expressions and rounding:
//   r~_j = r~_j - alpha s~_j,   s~_j = (d_j w_j - alpha (d_j u_j)) + beta s~_j
// (without a preconditioner s~ = s, r~ = r, d = 1). Those four vectors are
// double-buffered (second buffers P.b0 = s~ | s, P.b1 = r~ | r, P.b2 = w,
// P.p1 = u; set by ctrl->pcur); x, p (and r, s with Jacobi) are updated in
// place. The block SpMV runs before the step's checks are known, as in the
// reference. A breakdown of nu' keeps PprK1's partial update (w, w~ stored).
// streams: A, x p r s w u [s~ r~ d]
template <bool PREC>
struct PprF {
    static constexpr int NV = PREC ? 9 : 6, ND = 6;
    static constexpr int MAXNREG = CGVK_SPMV_MAXNREG;
    static constexpr bool CSR = true;
    static constexpr bool PDL_LATE = (CGVK_F_LATE & 4) != 0;
    static constexpr bool NO_BAND = true;
    static constexpr bool NO_PEER = true;
    static constexpr int STAGES = 2;
    static constexpr int MINB = 2;  // PprK1's register appetite
    static constexpr int SMEM_CTAS = 2;
    double alpha, beta, nup;
    bool valid, want_delta, want_dhat;
    const double *ac, *bc, *wc, *uc;  // inputs: a = s~ | s, b = r~ | r
    double *an, *bn, *wn, *un;        // outputs
    __device__ bool enter(const Params& P) {
        const Ctrl* c = P.ctrl;
        if (!step_wanted(c)) return false;
        alpha = c->sc[SA];
        nup = predicted_nu(P.nu_expr, c->sc);
        valid = isfinite(nup) && nup > 0.0;
        beta = DIV(nup, c->sc[SNU]);
        want_delta = P.nu_expr != 2 || P.track_delta;
        want_dhat = P.nu_expr == 0;
        double* const a0 = PREC ? P.st : P.s;
        double* const b0 = PREC ? P.rt : P.r;
        const bool b = c->pcur != 0;
        ac = b ? P.b0 : a0;
        an = b ? a0 : P.b0;
        bc = b ? P.b1 : b0;
        bn = b ? b0 : P.b1;
        wc = b ? P.b2 : P.w;
        wn = b ? P.w : P.b2;
        uc = b ? P.p1 : P.u;
        un = b ? P.u : P.p1;
        return true;
    }
    __device__ static bool entered(const Ctrl* c) { return PrF<PREC>::entered(c); }
    __device__ const double* vec(const Params& P, int v) const { return early_vec(P, v, wc == P.b2); }
    __device__ static const double* early_vec(const Params& P, int v, bool b) {
        const double* const a = b ? P.b0 : (PREC ? P.st : P.s);
        const double* const g = b ? P.b1 : (PREC ? P.rt : P.r);
        switch (v) {
            case 0: return P.x;
            case 1: return P.p0;
            case 2: return PREC ? P.r : g;
            case 3: return PREC ? P.s : a;
            case 4: return b ? P.b2 : P.w;
            case 5: return b ? P.p1 : P.u;
            case 6: return a;
            case 7: return g;
            default: return P.d;
        }
    }
    static constexpr int NG = PREC ? 5 : 4;
    __device__ const double* gsrc(const Params& P, int k) const {
        return k == 0 ? ac : k == 1 ? bc : k == 2 ? wc : k == 3 ? uc : P.d;
    }
    __device__ int sync() const { return 2; }
    __device__ unsigned int* counter(const Params& P) const { return &P.ctrl->count[1]; }
    template <class In, class RR>
    __device__ void row(const Params& P, int i, const In& in, const RR& R, double* acc) const {
        // PprK1's row
        const double p_old = SV(1), s_old = SV(3), w_old = SV(4), u = SV(5);
        P.x[i] = ADD(SV(0), MUL(alpha, p_old));
        const double r = SUB(SV(2), MUL(alpha, s_old));
        double rt = r, st_old = s_old;
        if constexpr (PREC) {
            P.r[i] = r;
            st_old = SV(6);
            rt = SUB(SV(7), MUL(alpha, st_old));
        }
        bn[i] = rt;
        const double wp = SUB(w_old, MUL(alpha, u));  // w'_k
        if (P.wpred) P.wpred[i] = wp;                  // run()'s probes track the prediction
        double wtp = wp;
        if constexpr (PREC) {
            const double d = SV(8);
            wtp = SUB(MUL(d, w_old), MUL(alpha, MUL(d, u)));
        }
        acc[5] = ADD(acc[5], MUL(r, r));
        if (!valid) {  // PprK1's breakdown step: w'_k (and w~'_k) stored, p, s, s~, u unchanged
            wn[i] = wp;
            if constexpr (PREC) P.wt[i] = wtp;
            an[i] = st_old;
            un[i] = u;
            return;
        }
        const double p = ADD(rt, MUL(beta, p_old));
        const double s = ADD(wp, MUL(beta, s_old));
        double st = s;
        if constexpr (PREC) {
            st = ADD(wtp, MUL(beta, st_old));
            P.s[i] = s;
        }
        an[i] = st;
        P.p0[i] = p;
        acc[0] = ADD(acc[0], MUL(p, s));
        if (want_delta) acc[1] = ADD(acc[1], MUL(rt, s));
        if (want_dhat) acc[2] = ADD(acc[2], MUL(st, r));
        acc[3] = ADD(acc[3], MUL(st, s));
        acc[4] = ADD(acc[4], MUL(rt, r));
        // PprK2's row: (u, w) = A (s~, r~), both re-formed at every gathered column
        const double* __restrict__ ag = ac;
        const double* __restrict__ bg = bc;
        const double* __restrict__ wg = wc;
        const double* __restrict__ ug = uc;
        const double* __restrict__ dg = P.d;
        const double a = alpha, b = beta;
        double un_, wn_;
        row_dot2(
            R,
            [=](int j) {
                const double so = in.gather(0, j, ag);
                const double wj = in.gather(2, j, wg), uj = in.gather(3, j, ug);
                double wt;
                if constexpr (PREC) {
                    const double dj = in.gather(4, j, dg);
                    wt = SUB(MUL(dj, wj), MUL(a, MUL(dj, uj)));
                } else {
                    wt = SUB(wj, MUL(a, uj));
                }
                return ADD(wt, MUL(b, so));
            },
            [=](int j) { return SUB(in.gather(1, j, bg), MUL(a, in.gather(0, j, ag))); }, un_, wn_);
        un[i] = un_;
        wn[i] = wn_;
    }
    __device__ void finish(const Params& P, Ctrl* c, const double* tot) const {
        c->pcur ^= 1;
        PprK1<PREC> k1;
        k1.alpha = alpha;
        k1.beta = beta;
        k1.nup = nup;
        k1.valid = valid;
        k1.want_delta = want_delta;
        k1.want_dhat = want_dhat;
        k1.recw = true;
        k1.finish(P, c, tot);
        c->mode2 = MODE_SKIP;  // (PprK2's finish: the block SpMV is done)
    }
};

// ============================================================  L1 SpMV
// y = A x (NRHS 1) or (y1, y2) = (A x1, A x2) in one pass (NRHS 2) through
// the solver's engines, for the C ABI's cgvk_spmv / cgvk_block_spmv
// (src/sparse_matrix.cpp:109-143): x1, x2 in P.w, P.u; y1, y2 in P.t, P.s.
// RESID: y = b - A x with b in P.u (initialize()'s r0, src/variants.cpp:376).
// Rows summed in CSR order, as every SpMV here.
template <int NRHS, bool RESID = false>
struct SpmvOp {
    static constexpr int NV = 0, ND = 0;
    static constexpr bool CSR = true;
    static constexpr int NG = NRHS;
    __device__ bool enter(const Params&) { return true; }
    __device__ const double* vec(const Params&, int) const { return nullptr; }
    __device__ const double* gsrc(const Params& P, int k) const { return k ? P.u : P.w; }
    __device__ int sync() const { return 0; }
    __device__ unsigned int* counter(const Params& P) const { return &P.ctrl->count[1]; }
    template <class In, class RR>
    __device__ void row(const Params& P, int i, const In& in, const RR& R, double*) const {
        const double* __restrict__ x1 = P.w;
        if constexpr (NRHS == 2) {
            const double* __restrict__ x2 = P.u;
            double y1, y2;
            row_dot2(R, [&](int j) { return in.gather(0, j, x1); }, [&](int j) { return in.gather(1, j, x2); }, y1,
                     y2);
            P.t[i] = y1;
            P.s[i] = y2;
        } else {
            const double y = row_dot(R, [&](int j) { return in.gather(0, j, x1); });
            P.t[i] = RESID ? SUB(P.u[i], y) : y;
        }
    }
    __device__ void finish(const Params&, Ctrl*, const double*) const {}
};

#undef SV

}  // namespace cgvk
