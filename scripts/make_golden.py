#!/usr/bin/env python3
"""Generate the committed golden fixtures under tests/golden/ from the
REFERENCE ITSELF (oracle/_ref/libcgvref.so: the unchanged reference sources,
built by oracle/Makefile). Run in the dev container, where /root/reference
exists; the GPU box only reads the outputs.

  mtx        tests/golden/mtx/<name>.npz — the 9 bundled Matrix-Market KAT
             matrices parsed by the reference parser (src/matrix_market.cpp)
             into the reference CSR layout.
  table3     tests/golden/table3.json — run() with the A-norm-error stop rule
             at 1e-5 (the Table-3 protocol, tests/test_matrices.cpp:39-46) for
             every fixture x {none, jacobi} x 7 variants, plus the fixed-budget
             min-log10-error cases of tests/test_matrices.cpp:86-111.
  small      tests/golden/small_traces.json — 25 reference steps on small
             synthetic problems, every scalar as a hex float, status and
             stats per step, and SHA-256 of every final vector.
  config     tests/golden/config_<name>.json — BASELINE configs: per variant
             the first 50 updated and true residual norms, iterations to
             ||r||/||b|| <= 1e-8, the final true residual.

  tree       tests/golden/tree_<name>.json — the same BASELINE configs through
             the C restatement in the B200's reduction order (ORC_DOT_TREE
             with the (block, gmax, order) cgvk_reduction_config reports on a
             148-SM B200): per variant the first 50 iterations' updated and
             true residual norms, alpha and beta as hex floats, and the
             measured distance of those norms from the reference's sequential
             ones (config_<name>.json) — the reorder floor.

Usage: make_golden.py mtx | table3 | small | config <name> [variant ...] | tree <name> [variant ...]
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_1905_01549_b200 import problems as pb  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")
MTX_DIR = "/root/reference/proj/data/matrices"
FIXTURES = ["1138_bus", "494_bus", "bcsstk03", "bcsstm21", "bcsstm22", "model_48_8_3", "nos2",
            "nos4", "nos7"]
VARIANT_IDS = {"hs": 0, "cg": 1, "m": 2, "pr": 3, "gv": 4, "pipe-pr-m": 5, "pipe-pr": 6}


def load_fixture(name: str) -> pb.CSR:
    d = np.load(os.path.join(GOLDEN, "mtx", name + ".npz"))
    return pb.CSR(int(d["n"]), d["row_ptr"], d["col_idx"], d["values"])


def cmd_mtx():
    os.makedirs(os.path.join(GOLDEN, "mtx"), exist_ok=True)
    for name in FIXTURES:
        m = O.ref_read_mtx(os.path.join(MTX_DIR, name + ".mtx"))
        n, rp, ci, va = m.arrays()
        np.savez_compressed(os.path.join(GOLDEN, "mtx", name + ".npz"), n=n, row_ptr=rp,
                            col_idx=ci, values=va)
        print(name, n, len(va))


def kat_problem(A: pb.CSR):
    # x* = 1/sqrt(n), b = A x*, x0 = 0 (tests/test_matrices.cpp:27-37)
    xs = np.full(A.n, 1.0 / np.sqrt(A.n))
    return xs, A.spmv(xs), np.zeros(A.n)


def cmd_table3():
    out = {"protocol": "run(), StopRule::error_reduction(1e-5), probes every iteration, "
                       "x*=1/sqrt(n), x0=0 (tests/test_matrices.cpp:39-46)", "runs": {}}
    for name in FIXTURES:
        A = load_fixture(name)
        xs, b, x0 = kat_problem(A)
        budget = 10 * A.n + 2000 if name != "nos2" else 40000
        for prec in (0, 1):
            for v, vid in VARIANT_IDS.items():
                t0 = time.time()
                r = O.ref_run(A, vid, prec, b, x0, xs, budget, 1, 1e-5, 1, 0)
                key = f"{name}/{'jacobi' if prec else 'none'}/{v}"
                out["runs"][key] = {"iters_to_1e5": r["iters_to_1e5"],
                                    "final_state": r["final_state"], "budget": budget}
                print(key, r["iters_to_1e5"], r["final_state"], f"{time.time() - t0:.1f}s")
    # fixed-budget attainable-accuracy cases (tests/test_matrices.cpp:86-111)
    fixed = {}
    for name, v, budget in [("bcsstk03", "pr", 1456), ("494_bus", "hs", 3592),
                            ("494_bus", "gv", 4200)]:
        A = load_fixture(name)
        xs, b, x0 = kat_problem(A)
        r = O.ref_run(A, VARIANT_IDS[v], 0, b, x0, xs, budget, 0, 1e-5, 1, 0)
        fixed[f"{name}/none/{v}"] = {"budget": budget, "iters_to_1e5": r["iters_to_1e5"],
                                     "min_log10_err": r["min_log10_err"]}
        print(name, v, r["iters_to_1e5"], r["min_log10_err"])
    out["fixed_budget"] = fixed
    with open(os.path.join(GOLDEN, "table3.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


SMALL = {
    "poisson3d_12": lambda: pb.poisson3d(12),
    "varcoef_10": lambda: pb.varcoef3d(10),
    "randspd_3000": lambda: pb.random_spd(3000, 13, 300, 7),
    "poisson2d_33": lambda: pb.poisson2d(33),
}
ABLATIONS = {
    "pr_meurant": (3, {"nu_expr": 2}),
    "pr_expanded": (3, {"nu_expr": 0}),
    "pr_no_recompute_nu": (3, {"recompute_nu": False}),
    "pipe_no_recompute_w": (6, {"recompute_w": False}),
    "pipe_expanded": (6, {"nu_expr": 0}),
    "m_track_delta": (2, {"track_delta": True}),
    "cg_unsimplified_mu": (1, {"unsimplified_mu": True}),
    "gv_unsimplified_mu": (4, {"unsimplified_mu": True}),
}


def hexs(d: dict) -> dict:
    return {k: float(v).hex() for k, v in d.items()}


def vec_hash(a) -> str | None:
    return None if a is None else hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def trace(solver, steps: int) -> dict:
    recs = []
    st = solver.state()
    recs.append({"k": st["k"], "state": st["state"], "breakdown": st["breakdown"],
                 "criterion": st["criterion"], "scalars": hexs(st["scalars"]), "stats": st["stats"],
                 "allocated_vectors": st["allocated_vectors"]})
    for _ in range(steps):
        if solver.state()["state"] != 0:
            break
        solver.step()
        st = solver.state()
        recs.append({"k": st["k"], "state": st["state"], "breakdown": st["breakdown"],
                     "criterion": st["criterion"], "scalars": hexs(st["scalars"]),
                     "stats": st["stats"]})
    vecs = {O.VEC_NAMES[w]: vec_hash(solver.vector(w)) for w in range(11)}
    return {"records": recs, "final_vectors_sha256": vecs}


def cmd_small():
    out = {"steps": 25, "cases": {}}
    for pname, make in SMALL.items():
        P = pb.make_problem(pname, make())
        for prec in (0, 1):
            for v, vid in VARIANT_IDS.items():
                s = O.Reference(P.A, vid, prec, P.b, P.x0)
                out["cases"][f"{pname}/{'jacobi' if prec else 'none'}/{v}"] = trace(s, 25)
            for ab, (vid, kw) in ABLATIONS.items():
                s = O.Reference(P.A, vid, prec, P.b, P.x0, **kw)
                out["cases"][f"{pname}/{'jacobi' if prec else 'none'}/{ab}"] = trace(s, 25)
        print(pname)
    out["ablations"] = {k: [v[0], v[1]] for k, v in ABLATIONS.items()}
    with open(os.path.join(GOLDEN, "small_traces.json"), "w") as f:
        json.dump(out, f, sort_keys=True)


def cmd_config(name: str, variants: list[str]):
    path = os.path.join(GOLDEN, f"config_{name}.json")
    data = json.load(open(path)) if os.path.exists(path) else {"config": name, "variants": {}}
    P = pb.config_problem(name)
    data.update({"n": P.A.n, "nnz": P.A.nnz, "precond": "jacobi", "tol": 1e-8,
                 "protocol": "reference initialize + step until ||r_k|| <= 1e-8 ||b|| "
                             "(sequential norm2, checked after each step); true residual "
                             "||b - A x_k|| from a fresh reference spmv for k <= 50"})
    for v in variants:
        t0 = time.time()
        s = O.Reference(P.A, VARIANT_IDS[v], 1, P.b, P.x0)
        taken, upd, tru = s.solve(P.b, 20000, 1e-8, true_cap=51)
        final_true = s.true_residual(P.b)
        st = s.state()
        data["variants"][v] = {"iters_to_1e-8": taken, "state": st["state"],
                               "upd_res_first51": [float(x).hex() for x in upd[:51]],
                               "true_res_first51": [float(x).hex() for x in tru[:51]],
                               "final_true_res": float(final_true).hex(),
                               "final_upd_res": float(upd[-1]).hex(),
                               "bnorm": float(np.sqrt(O.dot(P.b, P.b))).hex(),
                               "cpu_seconds": time.time() - t0}
        print(name, v, taken, final_true, f"{time.time() - t0:.1f}s", flush=True)
        # re-read before writing: several processes may fill one config
        cur = json.load(open(path)) if os.path.exists(path) else data
        cur.setdefault("variants", {})[v] = data["variants"][v]
        for k in ("config", "n", "nnz", "precond", "tol", "protocol"):
            cur[k] = data[k]
        with open(path + ".tmp", "w") as f:
            json.dump(cur, f, indent=1, sort_keys=True)
        os.replace(path + ".tmp", path)


# reduction tree of a 148-SM B200 per config (cgvk_reduction_config): the CSR
# engine G = 3 x SMs in strided tile order, the band engine (R4M) 6 x SMs in
# contiguous order
B200_TREE = {"p2d": (256, 444, 0), "p64": (256, 444, 0), "p128": (256, 444, 0), "v256": (256, 444, 0),
             "r4m": (256, 888, 1)}


def rel_dist(a, b) -> float:
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b) / np.abs(b)))


def cmd_tree(name: str, variants: list[str]):
    path = os.path.join(GOLDEN, f"tree_{name}.json")
    seq = json.load(open(os.path.join(GOLDEN, f"config_{name}.json")))
    P = pb.config_problem(name)
    block, gmax, order = B200_TREE[name]
    dot = ("tree", block, gmax, order)
    for v in variants:
        t0 = time.time()
        s = O.Restatement(P.A, VARIANT_IDS[v], 1, P.b, P.x0, dot=dot)

        def norms():
            r = s.vector(1)
            x = s.vector(0)
            e = P.b - O.spmv(P.A, x)
            return np.sqrt(O.dot(r, r, dot)), np.sqrt(O.dot(e, e, dot))

        upd, tru, alpha, beta = [], [], [], []
        u, t = norms()
        upd.append(u)
        tru.append(t)
        for _ in range(50):
            s.step()
            sc = s.state()["scalars"]
            alpha.append(sc["alpha"])
            beta.append(sc["beta"])
            u, t = norms()
            upd.append(u)
            tru.append(t)
        ref = seq["variants"][v]
        ref_upd = [float.fromhex(x) for x in ref["upd_res_first51"]]
        ref_tru = [float.fromhex(x) for x in ref["true_res_first51"]]
        rec = {"reduction": [block, gmax, order],
               "upd_res_first51": [float(x).hex() for x in upd],
               "true_res_first51": [float(x).hex() for x in tru],
               "alpha_1_50": [float(x).hex() for x in alpha],
               "beta_1_50": [float(x).hex() for x in beta],
               "floor_upd_vs_reference": rel_dist(upd, ref_upd),
               "floor_true_vs_reference": rel_dist(tru, ref_tru),
               "cpu_seconds": time.time() - t0}
        print(name, v, rec["floor_upd_vs_reference"], rec["floor_true_vs_reference"],
              f"{time.time() - t0:.1f}s", flush=True)
        cur = json.load(open(path)) if os.path.exists(path) else {"config": name, "variants": {}}
        cur["variants"][v] = rec
        cur.update({"n": P.A.n, "nnz": P.A.nnz, "precond": "jacobi",
                    "protocol": "C restatement (oracle/cgv_oracle.c) with ORC_DOT_TREE in the B200's "
                                "reduction order; norms of r_k and b - A x_k in that order; floor = max "
                                "relative distance of those norms from config_<name>.json (the reference)"})
        with open(path + ".tmp", "w") as f:
            json.dump(cur, f, indent=1, sort_keys=True)
        os.replace(path + ".tmp", path)


# run() with probes (proj/src/runner.cpp, proj/src/diagnostics.cpp): the
# reference's records for a few problems x variants x {none, Jacobi} x stop
# rules; oracle/run.py (seq order) must reproduce them, the device run() must
# match oracle/run.py in its own order (tests/test_run*.py).
RUN_CASES = [
    # (id, stop, cadence, probes, max_iter)
    ("fixed25", ("fixed", 25), 1, True, 60),
    ("error1e-6", ("error", 1e-6), 1, True, 200),
    ("stag5_c3", ("stagnation", 5, 0.01), 3, True, 80),
    ("noprobe_stag", ("stagnation", 4, 0.05), 1, False, 60),
]


def run_problems():
    return {"p2d_24": pb.make_problem("p2d_24", pb.poisson2d(24)),
            "rs_600": pb.make_problem("rs_600", pb.random_spd(600, 7, 90, 5))}


def cmd_run():
    out = {"fields": list(O.RECORD_FIELDS), "cases": {}}
    for pname, P in run_problems().items():
        for v in range(7):
            for prec in (0, 1):
                for cid, stop, cad, probes, mx in RUN_CASES:
                    r = O.ref_run_records(P.A, v, prec, P.b, P.x0, P.x_star, mx, stop, probes, cad)
                    key = f"{pname}/{v}/{prec}/{cid}"
                    out["cases"][key] = {
                        "problem": pname, "variant": v, "precond": prec, "stop": list(stop),
                        "cadence": cad, "probes": probes, "max_iter": mx,
                        "state": r["state"], "breakdown": r["breakdown"], "criterion": r["criterion"],
                        "summary": r["summary"],
                        "records": [[rec["k"]] + [None if rec[f] is None else float(rec[f]).hex()
                                                  for f in O.RECORD_FIELDS] for rec in r["records"]]}
    with open(os.path.join(GOLDEN, "run_records.json"), "w") as f:
        json.dump(out, f, sort_keys=True)
    print(len(out["cases"]), "run() cases")


if __name__ == "__main__":
    if not O.reference_available():
        sys.exit("oracle/_ref not built (make -C oracle ref)")
    cmd = sys.argv[1]
    if cmd == "mtx":
        cmd_mtx()
    elif cmd == "table3":
        cmd_table3()
    elif cmd == "small":
        cmd_small()
    elif cmd == "run":
        cmd_run()
    elif cmd == "config":
        cmd_config(sys.argv[2], sys.argv[3:] or ["hs", "cg", "m", "pr", "gv", "pipe-pr"])
    elif cmd == "tree":
        cmd_tree(sys.argv[2], sys.argv[3:] or ["hs", "cg", "m", "pr", "gv", "pipe-pr"])
    else:
        sys.exit(__doc__)
