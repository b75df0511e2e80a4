"""TEST INFRASTRUCTURE ONLY — restatement of the reference's run() driver with
its probes, on top of the C restatement stepper (oracle.Restatement).

Follows proj/src/runner.cpp:32-147 (loop, stop rules, cadence, residual
window) and proj/src/diagnostics.cpp:11-125 (probe, Lanczos three-term
residual, summarize) line by line. Vector arithmetic is elementwise numpy
(each product rounded before the add/subtract, as the reference's
-ffp-contract=off build); products use oracle.spmv (CSR row order) and
reductions use oracle.dot in the chosen order: "seq" reproduces the
reference itself (pinned against tests/golden/run_records.json, made by the
reference's own run()), ("tree", ...) reproduces the device's canonical order.
"""
from __future__ import annotations

import math

import numpy as np

from . import oracle as O

X, R, P, S, W, U = 0, 1, 2, 3, 4, 5
R_TILDE = 7
RUNNING = 0
MAX_ITERATIONS, CONVERGED = 2, 3
ERROR_THRESHOLD, STAGNATION = 1, 2
PREDICTORS = (2, 3, 5, 6)  # M, PR, PIPE_PR_M, PIPE_PR
PIPELINED = (4, 5, 6)      # GV, PIPE_PR_M, PIPE_PR
GV = 4


def _norm(x, mode):  # norm2, inc/vector_ops.hpp:27-29
    return math.sqrt(O.dot(x, x, mode))


def _a_norm(A, e, mode):  # src/sparse_matrix.cpp:169-178
    q = O.dot(e, O.spmv(A, e), mode)
    return math.sqrt(max(q, 0.0))


def probe(o, A, b, precond, variant, cfg, mode, x_star=None, e0=0.0, prev_r=None, w_pred=None):
    """src/diagnostics.cpp:11-72 on the restatement's current state."""
    st = o.state()
    sc = st["scalars"]
    k = st["k"]
    x, r = o.vector(X), o.vector(R)
    rec = {"k": k}
    ax = O.spmv(A, x)
    true_res = b - ax
    rec["true_res_norm"] = _norm(true_res, mode)
    rec["upd_res_norm"] = _norm(r, mode)
    rec["residual_gap_norm"] = _norm(true_res - r, mode)
    if x_star is not None:
        rec["rel_err_a_norm"] = _a_norm(A, x_star - x, mode) / e0
    rt = o.vector(R_TILDE) if precond else r
    if variant in PREDICTORS and k >= 1:
        rec["nu_gap"] = O.dot(rt, r, mode) - sc["nu_prime"]
        rec["nu_prime"] = sc["nu_prime"]
    if variant in PIPELINED:
        if variant == GV or not cfg.get("recompute_w", True) or k == 0:
            wp = o.vector(W)
        else:
            wp = w_pred
        if wp is not None:
            rec["w_gap_norm"] = _norm(O.spmv(A, rt) - wp, mode)
        rec["s_gap_norm"] = _norm(O.spmv(A, o.vector(P)) - o.vector(S), mode)
    if prev_r is not None and k >= 1:
        nr, np_ = _norm(r, mode), _norm(prev_r, mode)
        if nr > 0.0 and np_ > 0.0:
            rec["succ_orth"] = O.dot(r, prev_r, mode) / (nr * np_)
    rec["alpha"] = sc["alpha"]
    if k >= 1:
        rec["beta"] = sc["beta"]
    rec["nu"] = sc["nu"]
    return rec


def lanczos(A, r_km2, r_km1, r_k, a_km2, a_km1, b_km1, k, mode):
    """src/diagnostics.cpp:74-109."""
    n_k, n_km1, n_km2 = _norm(r_k, mode), _norm(r_km1, mode), _norm(r_km2, mode)
    sign_kp1 = 1.0 if k % 2 == 0 else -1.0
    sign_k, sign_km1 = -sign_kp1, sign_kp1
    q_k = sign_k * r_km1 / n_km1
    lhs = O.spmv(A, q_k)
    c_kp1 = (1.0 / a_km1) * (n_k / n_km1)
    c_k = 1.0 / a_km1 + b_km1 / a_km2
    c_km1 = (1.0 / a_km2) * (n_km1 / n_km2)
    q_kp1 = sign_kp1 * r_k / n_k
    q_km1 = sign_km1 * r_km2 / n_km2
    d = lhs - (c_kp1 * q_kp1 + c_k * q_k + c_km1 * q_km1)
    return math.sqrt(O.dot(d, d, mode))


def run(A, variant: int, precond: int, b, x0, max_iter: int, stop=("stagnation", 50, 0.01),
        probes: bool = True, cadence: int = 1, x_star=None, mode="seq", **cfg) -> dict:
    """src/runner.cpp:32-147. stop: ("fixed", n) | ("error", thr) | ("stagnation", window, impr).
    cfg: nu_expr, recompute_nu, recompute_w, unsimplified_mu, track_delta."""
    if max_iter < 0:
        raise ValueError("max_iter must be >= 0")
    if stop[0] == "error" and x_star is None:
        raise ValueError("error-reduction stop rule needs x*")
    b, x0 = np.asarray(b, np.float64), np.asarray(x0, np.float64)
    o = O.Restatement(A, variant, precond, b, x0, dot=mode, **cfg)
    track = variant in PIPELINED and probes and cfg.get("recompute_w", True) and variant != GV
    e0 = 0.0
    if x_star is not None:
        x_star = np.asarray(x_star, np.float64)
        e0 = _a_norm(A, x_star - x0, mode)
        if e0 == 0.0:
            raise ValueError("x0 already equals x*; error ratios undefined")
    cadence = cadence if cadence >= 1 else 1
    records = []
    w_pred = None
    if probes:
        records.append(probe(o, A, b, precond, variant, cfg, mode, x_star, e0))
    win = {"r_km1": o.vector(R), "r_km2": None, "a_km1": o.state()["scalars"]["alpha"], "a_km2": 0.0,
           "b_km1": 0.0, "filled": 1}

    def push(r, alpha, beta):
        win["r_km2"], win["a_km2"] = win["r_km1"], win["a_km1"]
        win["r_km1"], win["a_km1"], win["b_km1"] = r, alpha, beta
        win["filled"] = min(win["filled"] + 1, 2)

    best = records[0].get("true_res_norm", 0.0) if records else 0.0
    if not probes:
        best = _norm(b - O.spmv(A, o.vector(X)), mode)
    last_k = 0
    budget = min(max_iter, stop[1]) if stop[0] == "fixed" else max_iter
    final = None
    while o.state()["state"] == RUNNING and o.state()["k"] < budget:
        if track:  # w'_k = w_{k-1} - alpha u_{k-1} (src/variants.cpp:310-312)
            w_prev, u_prev = o.vector(W), o.vector(U)
            w_pred = w_prev - o.state()["scalars"]["alpha"] * u_prev
        o.step()
        st = o.state()
        terminal = st["state"] != RUNNING
        k = st["k"]
        err = tres = None
        if stop[0] == "error":
            err = _a_norm(A, x_star - o.vector(X), mode) / e0
        elif stop[0] == "stagnation":
            tres = _norm(b - O.spmv(A, o.vector(X)), mode)
        stop_now, stop_status = False, None
        if err is not None and err < stop[1]:
            stop_now, stop_status = True, (CONVERGED, 0, ERROR_THRESHOLD)
        if tres is not None:
            if tres < best * (1.0 - stop[2]):
                best, last_k = tres, k
            elif k - last_k >= stop[1]:
                stop_now, stop_status = True, (CONVERGED, 0, STAGNATION)
        if probes and (terminal or stop_now or k % cadence == 0):
            rec = probe(o, A, b, precond, variant, cfg, mode, x_star, e0,
                        win["r_km1"] if win["filled"] >= 1 else None, w_pred)
            if (win["filled"] >= 2 and rec.get("upd_res_norm", 0.0) > 0.0
                    and _norm(win["r_km1"], mode) > 0.0 and _norm(win["r_km2"], mode) > 0.0
                    and win["a_km1"] != 0.0 and win["a_km2"] != 0.0):
                rec["lanczos_res_norm"] = lanczos(A, win["r_km2"], win["r_km1"], o.vector(R),
                                                  win["a_km2"], win["a_km1"], win["b_km1"], k, mode)
            records.append(rec)
        push(o.vector(R), st["scalars"]["alpha"], st["scalars"]["beta"])
        if stop_now and not terminal:
            final = stop_status
            break
    if final is None:
        st = o.state()
        final = (MAX_ITERATIONS if st["state"] == RUNNING else st["state"], st["breakdown"],
                 st["criterion"])
    summary = None
    ratios = [(r["k"], r["rel_err_a_norm"]) for r in records if "rel_err_a_norm" in r]
    if probes and x_star is not None and ratios:  # summarize, src/diagnostics.cpp:111-125
        first = next((k for k, q in ratios if q < 1e-5), None)
        summary = {"iters_to_1e5": first, "min_log10_err": math.log10(min(q for _, q in ratios))}
    full = [{f: rec.get(f) for f in ("k",) + O.RECORD_FIELDS} for rec in records]
    return {"state": final[0], "breakdown": final[1], "criterion": final[2], "records": full,
            "summary": summary, "x": o.vector(X)}
