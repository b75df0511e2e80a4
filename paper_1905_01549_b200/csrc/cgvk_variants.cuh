// The per-iteration kernels of the six CG variants (+ pipe-PR-M, M via the
// nu' expression), as fused two-kernel schedules.
//
// Each iteration is exactly two launches, K1 then K2, captured in a CUDA
// graph. Global reductions are folded by the last-arriving CTA of the kernel
// that produces the operands, which also runs the scalar recurrences and the
// breakdown/convergence checks of src/variants.cpp:128-187 on the device, so
// the host never synchronises inside the loop. Every vector value is bit-
// identical to the reference's (no FMA; the Jacobi products d∘v that the
// reference stores are recomputed on the fly from the same operands); dots
// follow the canonical tree of cgvk_device.cuh.
//
// After K1/K2 of step k the device holds the reference state after step(k)
// (src/variants.cpp:446-458) except for the beta-recurrences that CG-CG and GV
// defer into the next K1 (`form_pending`); the host materialises them (a K1
// launch with k_limit = k) before reading vectors. Terminal steps keep the
// reference's partial-update semantics through `mode2` / `form_pending`.
#pragma once

#include "cgvk_device.cuh"

namespace cgvk {

template <bool PREC>
__device__ __forceinline__ double M_(const Params& P, int i, double v) {
    if constexpr (PREC) return MUL(__ldg(P.d + i), v);
    return v;
}

__device__ __forceinline__ bool step_wanted(const Ctrl* c) {
    return c->state == ST_RUNNING && c->k < c->k_limit;
}

#define TILE_LOOP(P)                                                                   \
    for (int tile = blockIdx.x; tile < (P).ntiles; tile += gridDim.x)                  \
        if (const int i = tile * kBlock + threadIdx.x; i < (P).n)

// =====================================================================  HS
// src/variants.cpp:189-205, paper Alg. 1. V = 3+1 (K1) + 4+3 (K2) vectors.

// K1: r -= alpha*s; nu = <M r, r>, <r,r>
template <bool PREC>
__global__ void __launch_bounds__(kBlock, kMinBlocksPerSM) hs_k1(Params P) {
    Ctrl* c = P.ctrl;
    if (!step_wanted(c)) return;
    const double alpha = c->sc[SA];
    double acc[2] = {0.0, 0.0}, tot[2];
    TILE_LOOP(P) {
        const double r = SUB(P.r[i], MUL(alpha, P.s[i]));
        P.r[i] = r;
        acc[0] = ADD(acc[0], MUL(M_<PREC>(P, i, r), r));
        acc[1] = ADD(acc[1], MUL(r, r));
    }
    if (!reduce_grid<2>(acc, P.part, &c->count[0], tot)) return;
    if (threadIdx.x != 0) return;
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

// K2: x += alpha*p_old; p = M r + beta p_old (on the fly for every gathered
// column); s = A p; mu = <p,s>
template <bool PREC>
__global__ void __launch_bounds__(kBlock, kMinBlocksPerSM) hs_k2(Params P) {
    Ctrl* c = P.ctrl;
    const int mode = c->mode2;
    if (mode == MODE_SKIP) return;
    const int pc = c->pcur;
    const double* __restrict__ pold = pc ? P.p1 : P.p0;
    double* pnew = pc ? P.p0 : P.p1;
    const double alpha = c->sc[SA], beta = c->sc[SB];
    const double* __restrict__ r = P.r;
    double acc[1] = {0.0}, tot[1];
    TILE_LOOP(P) {
        const double po = pold[i];
        P.x[i] = ADD(P.x[i], MUL(alpha, po));
        if (mode == MODE_FULL) {
            const double sum = row_sum(P, i, [&](int j) {
                return ADD(M_<PREC>(P, j, __ldg(r + j)), MUL(beta, __ldg(pold + j)));
            });
            const double pi = ADD(M_<PREC>(P, i, r[i]), MUL(beta, po));
            pnew[i] = pi;
            P.s[i] = sum;
            acc[0] = ADD(acc[0], MUL(pi, sum));
        }
    }
    if (!reduce_grid<1>(acc, P.part, &c->count[1], tot)) return;
    if (threadIdx.x != 0) return;
    c->mode2 = MODE_SKIP;
    if (mode != MODE_FULL) return;
    c->pcur = pc ^ 1;
    c->stats[STAT_SPMV] += 1;
    c->stats[STAT_RED] += 1;
    c->sc[SMU] = tot[0];
    if (settle_mu(c)) return;
    if (finalize_alpha(c)) return;
    check_tolerance(c);
}

// ==================================================================  CG-CG
// src/variants.cpp:207-234. K1 = tail of step k-1 (p, s recurrences) + head
// of step k (x, r); K2 = w = A M r with nu, eta (+ unsimplified dots).

template <bool PREC>
__global__ void __launch_bounds__(kBlock, kMinBlocksPerSM) cg_k1(Params P) {
    Ctrl* c = P.ctrl;
    const bool F = c->form_pending != 0, S = step_wanted(c);
    if (!F && !S) return;
    const double alpha = c->sc[SA], beta = c->sc[SB];
    TILE_LOOP(P) {
        double p = P.p0[i], s = P.s[i];
        if (F) {
            p = ADD(M_<PREC>(P, i, P.r[i]), MUL(beta, p));
            s = ADD(P.w[i], MUL(beta, s));
            P.p0[i] = p;
            P.s[i] = s;
        }
        if (S) {
            P.x[i] = ADD(P.x[i], MUL(alpha, p));
            P.r[i] = SUB(P.r[i], MUL(alpha, s));
        }
    }
    if (F && !S) {  // materialisation only: clear the debt
        if (arrive_last(&c->count[0]) && threadIdx.x == 0) {
            c->form_pending = 0;
            c->count[0] = 0u;
        }
    }
}

template <bool PREC>
__global__ void __launch_bounds__(kBlock, kMinBlocksPerSM) cg_k2(Params P) {
    Ctrl* c = P.ctrl;
    if (!step_wanted(c)) return;
    const bool unsimp = P.unsimplified_mu != 0;
    const double* __restrict__ r = P.r;
    double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0}, tot[5];
    TILE_LOOP(P) {
        const double w = row_sum(P, i, [&](int j) { return M_<PREC>(P, j, __ldg(r + j)); });
        P.w[i] = w;
        const double ri = r[i], rti = M_<PREC>(P, i, ri);
        acc[0] = ADD(acc[0], MUL(rti, ri));
        acc[1] = ADD(acc[1], MUL(rti, w));
        acc[2] = ADD(acc[2], MUL(ri, ri));
        if (unsimp) {
            acc[3] = ADD(acc[3], MUL(rti, P.s[i]));   // <r~_k, s_{k-1}>
            acc[4] = ADD(acc[4], MUL(P.p0[i], w));     // <p_{k-1}, w_k>
        }
    }
    if (!reduce_grid<5>(acc, P.part, &c->count[1], tot)) return;
    if (threadIdx.x != 0) return;
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

// ===============================================================  PR / M
// src/variants.cpp:237-265, paper Alg. 2 (M-CG with the Meurant nu').
// K1: x, r, r~ (s~ = M s on the fly) and p; K2: s = A p with mu, delta,
// delta-hat, gamma (s~ on the fly), nu, <r,r>.

template <bool PREC>
__global__ void __launch_bounds__(kBlock, kMinBlocksPerSM) pr_k1(Params P) {
    Ctrl* c = P.ctrl;
    if (!step_wanted(c)) return;
    const double alpha = c->sc[SA];
    const double nup = predicted_nu(P.nu_expr, c->sc);
    const bool valid = isfinite(nup) && nup > 0.0;
    const double beta = DIV(nup, c->sc[SNU]);
    double acc[1] = {0.0}, tot[1];
    TILE_LOOP(P) {
        const double s = P.s[i];
        P.x[i] = ADD(P.x[i], MUL(alpha, P.p0[i]));
        const double r = SUB(P.r[i], MUL(alpha, s));
        P.r[i] = r;
        double rt = r;
        if constexpr (PREC) {
            rt = SUB(P.rt[i], MUL(alpha, M_<PREC>(P, i, s)));
            P.rt[i] = rt;
        }
        if (valid)
            P.p0[i] = ADD(rt, MUL(beta, P.p0[i]));
        else
            acc[0] = ADD(acc[0], MUL(r, r));
    }
    if (valid) return;  // K2 finishes the step
    if (!reduce_grid<1>(acc, P.part, &c->count[0], tot)) return;
    if (threadIdx.x != 0) return;
    c->k += 1;
    c->sc[SNUP] = nup;
    record_rr(P, c, tot[0]);
    settle_nonpositive(c, nup, BR_NUPRIME, tot[0]);
}

template <bool PREC>
__global__ void __launch_bounds__(kBlock, kMinBlocksPerSM) pr_k2(Params P) {
    Ctrl* c = P.ctrl;
    if (!step_wanted(c)) return;
    const double nup = predicted_nu(P.nu_expr, c->sc);
    if (!(isfinite(nup) && nup > 0.0)) return;
    const bool want_delta = P.nu_expr != 2 || P.track_delta;
    const bool want_dhat = P.nu_expr == 0;
    const double* __restrict__ p = P.p0;
    double acc[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0}, tot[6];
    TILE_LOOP(P) {
        const double s = row_sum(P, i, [&](int j) { return __ldg(p + j); });
        P.s[i] = s;
        const double st = M_<PREC>(P, i, s);
        const double r = P.r[i];
        const double rt = PREC ? P.rt[i] : r;
        acc[0] = ADD(acc[0], MUL(p[i], s));
        if (want_delta) acc[1] = ADD(acc[1], MUL(rt, s));
        if (want_dhat) acc[2] = ADD(acc[2], MUL(st, r));
        acc[3] = ADD(acc[3], MUL(st, s));
        acc[4] = ADD(acc[4], MUL(rt, r));
        acc[5] = ADD(acc[5], MUL(r, r));
    }
    if (!reduce_grid<6>(acc, P.part, &c->count[1], tot)) return;
    if (threadIdx.x != 0) return;
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

// ====================================================================  GV
// src/variants.cpp:267-298. K1 = beta-recurrences of step k-1 (p, s, s~, u)
// + step k updates (x, r, r~, w) with nu, eta; the reduction is folded at
// the end of K1, so on multi-GPU it overlaps K2 = t = A M w.

template <bool PREC>
__global__ void __launch_bounds__(kBlock, kMinBlocksPerSM) gv_k1(Params P) {
    Ctrl* c = P.ctrl;
    const bool F = c->form_pending != 0, S = step_wanted(c);
    if (!F && !S) return;
    const double alpha = c->sc[SA], beta = c->sc[SB];
    const bool unsimp = P.unsimplified_mu != 0;
    double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0}, tot[5];
    TILE_LOOP(P) {
        double p = P.p0[i], s = P.s[i], u = P.u[i], w = P.w[i];
        double st = PREC ? P.st[i] : s;
        double rt = PREC ? P.rt[i] : P.r[i];
        if (F) {
            p = ADD(rt, MUL(beta, p));
            s = ADD(w, MUL(beta, s));
            if constexpr (PREC) st = ADD(M_<PREC>(P, i, w), MUL(beta, st));
            else st = s;
            u = ADD(P.t[i], MUL(beta, u));
            P.p0[i] = p;
            P.s[i] = s;
            if constexpr (PREC) P.st[i] = st;
            P.u[i] = u;
        }
        if (S) {
            P.x[i] = ADD(P.x[i], MUL(alpha, p));
            const double r = SUB(P.r[i], MUL(alpha, s));
            P.r[i] = r;
            if constexpr (PREC) {
                rt = SUB(rt, MUL(alpha, st));
                P.rt[i] = rt;
            } else {
                rt = r;
            }
            w = SUB(w, MUL(alpha, u));
            P.w[i] = w;
            acc[0] = ADD(acc[0], MUL(rt, r));
            acc[1] = ADD(acc[1], MUL(rt, w));
            acc[2] = ADD(acc[2], MUL(r, r));
            if (unsimp) {
                acc[3] = ADD(acc[3], MUL(rt, s));  // <r~_k, s_{k-1}>
                acc[4] = ADD(acc[4], MUL(p, w));   // <p_{k-1}, w_k>
            }
        }
    }
    if (!S) {  // materialisation only
        if (arrive_last(&c->count[0]) && threadIdx.x == 0) {
            c->form_pending = 0;
            c->count[0] = 0u;
        }
        return;
    }
    if (!reduce_grid<5>(acc, P.part, &c->count[0], tot)) return;
    if (threadIdx.x != 0) return;
    c->k += 1;
    c->mode2 = MODE_FULL;  // t = A w~ precedes the checks in the reference
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

template <bool PREC>
__global__ void __launch_bounds__(kBlock, kMinBlocksPerSM) gv_k2(Params P) {
    Ctrl* c = P.ctrl;
    if (c->mode2 == MODE_SKIP) return;
    const double* __restrict__ w = P.w;
    TILE_LOOP(P) {
        P.t[i] = row_sum(P, i, [&](int j) { return M_<PREC>(P, j, __ldg(w + j)); });
    }
    if (arrive_last(&c->count[1]) && threadIdx.x == 0) {
        c->mode2 = MODE_SKIP;
        c->count[1] = 0u;
    }
}

// ===============================================================  pipe-PR
// src/variants.cpp:303-350, paper Alg. 3 and the §2.2.1 schedule
// (PAPER.md:384-401): every dot of step k is computed in K1 from the updated
// vectors (they do not depend on u, w), so its reduction overlaps the block
// SpMV K2 = (u, w) = A (s~, r~). w~ = M w and u~ = M u are recomputed on the
// fly (recompute_w); with recompute_w off, w and w~ are stored recurrences.

template <bool PREC>
__global__ void __launch_bounds__(kBlock, kMinBlocksPerSM) ppr_k1(Params P) {
    Ctrl* c = P.ctrl;
    if (!step_wanted(c)) return;
    const double alpha = c->sc[SA];
    const double nup = predicted_nu(P.nu_expr, c->sc);
    const bool valid = isfinite(nup) && nup > 0.0;
    const double beta = DIV(nup, c->sc[SNU]);
    const bool want_delta = P.nu_expr != 2 || P.track_delta;
    const bool want_dhat = P.nu_expr == 0;
    const bool recw = P.recompute_w != 0;
    double acc[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0}, tot[6];
    TILE_LOOP(P) {
        P.x[i] = ADD(P.x[i], MUL(alpha, P.p0[i]));
        const double s_old = P.s[i];
        const double r = SUB(P.r[i], MUL(alpha, s_old));
        P.r[i] = r;
        double rt = r, st_old = s_old;
        if constexpr (PREC) {
            st_old = P.st[i];
            rt = SUB(P.rt[i], MUL(alpha, st_old));
            P.rt[i] = rt;
        }
        const double u = P.u[i];
        const double wn = SUB(P.w[i], MUL(alpha, u));  // w'_k
        double wtn = wn;
        if constexpr (PREC) {
            const double wt_old = recw ? M_<PREC>(P, i, P.w[i]) : P.wt[i];
            wtn = SUB(wt_old, MUL(alpha, M_<PREC>(P, i, u)));
        }
        if (valid) {
            const double p = ADD(rt, MUL(beta, P.p0[i]));
            const double s = ADD(wn, MUL(beta, s_old));
            double st = s;
            if constexpr (PREC) {
                st = ADD(wtn, MUL(beta, st_old));
                P.st[i] = st;
            }
            P.p0[i] = p;
            P.s[i] = s;
            if (!recw) {
                P.w[i] = wn;
                if constexpr (PREC) P.wt[i] = wtn;
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
    if (!reduce_grid<6>(acc, P.part, &c->count[0], tot)) return;
    if (threadIdx.x != 0) return;
    c->k += 1;
    c->sc[SNUP] = nup;
    record_rr(P, c, tot[5]);
    if (!valid) {
        c->wt_stored = PREC;
        settle_nonpositive(c, nup, BR_NUPRIME, tot[5]);
        return;
    }
    c->sc[SB] = beta;
    c->mode2 = MODE_FULL;  // the block SpMV precedes the checks in the reference
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

template <bool PREC>
__global__ void __launch_bounds__(kBlock, kMinBlocksPerSM) ppr_k2(Params P) {
    Ctrl* c = P.ctrl;
    if (c->mode2 == MODE_SKIP) return;
    const double* __restrict__ sv = PREC ? P.st : P.s;
    const double* __restrict__ rv = PREC ? P.rt : P.r;
    if (P.recompute_w) {
        TILE_LOOP(P) {
            double u, w;
            row_sum2(P, i, [&](int j) { return __ldg(sv + j); }, [&](int j) { return __ldg(rv + j); },
                     u, w);
            P.u[i] = u;
            P.w[i] = w;
        }
    } else {
        TILE_LOOP(P) { P.u[i] = row_sum(P, i, [&](int j) { return __ldg(sv + j); }); }
    }
    if (arrive_last(&c->count[1]) && threadIdx.x == 0) {
        c->mode2 = MODE_SKIP;
        c->count[1] = 0u;
    }
}

#undef TILE_LOOP

}  // namespace cgvk
