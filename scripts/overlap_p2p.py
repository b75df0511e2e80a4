"""Measured overlap of the reductions with the SpMV (north star: "measured
overlap of reductions/halo with SpMV for the pipelined and PR variants").

One GPU per call here, so the link latency is injected: a one-rank
peer-memory group (CGVK_GROUP_P2P; the same kernels, chained schedule and
in-kernel total exchange as a multi-GPU rank) where a published rank total
counts as arrived only CGVK_P2P_DELAY_NS after its publication. Each
variant's time per iteration is measured for several injected latencies L;
its slope d(t_iter)/dL is the number of reductions per iteration the variant
leaves exposed — Table 1 of the paper (src/cost_model.cpp:
15-30): HS 2 (C_gr twice), CG-CG / M / PR 1, GV and pipe-PR 0 up to the SpMV
time (max(C_gr, T_mv + C_mv)).

usage: python scripts/overlap_p2p.py [configs...] > profiles/r02/overlap_p2p.md
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_1905_01549_b200 import cgvk, problems as pb  # noqa: E402
from paper_1905_01549_b200.cgvk import Precond, Variant, VariantConfig  # noqa: E402

VARIANTS = [Variant.HS, Variant.CG_CG, Variant.M, Variant.PR, Variant.GV, Variant.PIPE_PR]
DELAYS_US = [0, 2, 5, 10, 20]
ITERS = {"p64": 400, "p128": 200}
ALIGN = {"p64": 64 * 64, "p128": 128 * 128}


def us_per_iter(P, cfg, v, delay_us, iters):
    os.environ["CGVK_P2P_DELAY_NS"] = str(int(delay_us * 1000))
    A = P.A
    lo = cgvk.partition_rows(A.n, 1, ALIGN[cfg])
    mats = [cgvk.RankMatrix(A.n, lo, 0, *cgvk.local_rows(A, lo, 0))]
    comm = cgvk.Comm(1)
    g = cgvk.Group(comm, mats, VariantConfig.make(v), Precond.JACOBI, [P.b], [P.x0], p2p=True)
    assert g.transport == "p2p"
    s = g.solvers[0]
    s.time_steps(5)
    ms, it = s.time_steps(iters)
    g.sync()
    hist = s.history()
    g.close()
    mats[0].close()
    comm.close()
    return 1e3 * ms / max(it, 1), hist


def main(configs):
    out = {}
    print("# Measured reduction / SpMV overlap (round 2)\n")
    print(__doc__.split("usage:")[0].strip().replace("\n", " ") + "\n")
    for cfg in configs:
        P = pb.config_problem(cfg)
        rows = {}
        for v in VARIANTS:
            t, ref = [], None
            for d in DELAYS_US:
                us, hist = us_per_iter(P, cfg, v, d, ITERS[cfg])
                if ref is None:
                    ref = hist
                assert np.array_equal(hist.view(np.int64), ref.view(np.int64))  # same bits at any latency
                t.append(us)
            slope = float(np.polyfit(DELAYS_US, t, 1)[0])
            rows[v.name] = {"us_per_iter": t, "slope": slope}
        out[cfg] = rows
        print(f"## {cfg}\n")
        print("| variant | " + " | ".join(f"L = {d} us" for d in DELAYS_US) + " | exposed reductions (slope) |")
        print("|---|" + "---:|" * (len(DELAYS_US) + 1))
        for name, r in rows.items():
            print(f"| {name} | " + " | ".join(f"{x:.1f}" for x in r["us_per_iter"]) + f" | {r['slope']:.2f} |")
        print()
    os.environ.pop("CGVK_P2P_DELAY_NS", None)
    print("```json")
    print(json.dumps(out, indent=1))
    print("```")


if __name__ == "__main__":
    main(sys.argv[1:] or ["p64", "p128"])
