"""Multi-GPU cost-model calibration from measured components (SURVEY §8(f)4,
the reference's src/cost_model.cpp: Table 1, max(C_gr, T_mv + C_mv) for the
pipelined variants, C_gr + T_mv + C_mv for the others).

One GPU per call here, so the P-rank solve runs as P in-process ranks with
the peer-memory transport (CGVK_GROUP_P2P) on one device: every kernel of
every rank is serialised on one stream, so the measured time per iteration / P
is the per-rank compute cost T_rank(P) — both kernels, their fills, tails and
the in-kernel exchange work — with every wait already satisfied. The
network term is the one thing not measurable here: a peer store lands in
L_nv ~ 1 us (half of the 1834-cycle peer-load round trip of the
microarchitecture guide), and each iteration exposes it once per reduction
the variant waits for (HS 2, CG-CG 1, M / PR 1, GV 0, pipe-PR 0: GV's and
pipe-PR's K1 reduction is folded by the next K1, behind the SpMV and its
halo). The predicted P-GPU time per iteration is T_rank(P) + n_exposed * L_nv,
shown for L_nv = 1 and 2 us next to the measured single-GPU time.

usage: python scripts/cost_model_ranks.py [configs...] > profiles/r02/cost_model.md
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1905_01549_b200 import cgvk, problems as pb  # noqa: E402
from paper_1905_01549_b200.cgvk import Precond, Variant, VariantConfig  # noqa: E402

VARIANTS = [Variant.HS, Variant.CG_CG, Variant.M, Variant.PR, Variant.GV, Variant.PIPE_PR]
EXPOSED = {Variant.HS: 2, Variant.CG_CG: 1, Variant.M: 1, Variant.PR: 1, Variant.GV: 0, Variant.PIPE_PR: 0}
PLANE = {"p64": 64 * 64, "p128": 128 * 128, "v256": 256 * 256}
ITERS = {"p64": 400, "p128": 200, "v256": 40}


def time_single(P, v, iters):
    A = cgvk.DeviceMatrix.from_csr(P.A)
    s = cgvk.initialize(VariantConfig.make(v), A, Precond.JACOBI, P.b, P.x0)
    s.time_steps(5)
    ms, it = s.time_steps(iters)
    s.close()
    A.close()
    return 1e3 * ms / max(it, 1)


def time_ranks(P, v, nranks, plane, iters):
    A = P.A
    lo = cgvk.partition_rows(A.n, nranks, plane)
    mats = [cgvk.RankMatrix(A.n, lo, r, *cgvk.local_rows(A, lo, r)) for r in range(nranks)]
    comm = cgvk.Comm(nranks)
    g = cgvk.Group(comm, mats, VariantConfig.make(v), Precond.JACOBI,
                   [P.b[lo[r]:lo[r + 1]] for r in range(nranks)], [P.x0[lo[r]:lo[r + 1]] for r in range(nranks)],
                   p2p=True)
    assert g.transport == "p2p"
    s = g.solvers[0]
    s.time_steps(5)
    ms, it = s.time_steps(iters)
    g.sync()
    g.close()
    for m in mats:
        m.close()
    comm.close()
    return 1e3 * ms / max(it, 1) / nranks


def main(configs):
    out = {}
    print("# Multi-GPU cost model from measured components (round 2)\n")
    print(__doc__.split("usage:")[0].strip().replace("\n", " ") + "\n")
    for cfg in configs:
        P = pb.config_problem(cfg)
        iters = ITERS.get(cfg, 100)
        rows = {}
        for v in VARIANTS:
            one = time_single(P, v, iters)
            per = {n: time_ranks(P, v, n, PLANE[cfg], iters) for n in (2, 4, 8)}
            rows[v.name] = {"single_gpu_us": one, "t_rank_us": per, "exposed": EXPOSED[v]}
        out[cfg] = rows
        print(f"## {cfg} (n = {P.A.n:,}, nnz = {P.A.nnz:,})\n")
        print("| variant | 1 GPU us/iter (measured) | T_rank us @2,4,8 (measured) | exposed waits | "
              "predicted us/iter @2,4,8, L_nv = 1 us | @8, L_nv = 2 us | speed-up @8 (L_nv = 1) |")
        print("|---|---:|---|---:|---|---:|---:|")
        for name, r in rows.items():
            e = r["exposed"]
            t = r["t_rank_us"]
            pred = {n: t[n] + e * 1.0 for n in t}
            print(f"| {name} | {r['single_gpu_us']:.1f} | {', '.join(f'{t[n]:.1f}' for n in (2, 4, 8))} | {e} | "
                  f"{', '.join(f'{pred[n]:.1f}' for n in (2, 4, 8))} | {t[8] + 2.0 * e:.1f} | "
                  f"{r['single_gpu_us'] / pred[8]:.2f} |")
        print()
    print("```json")
    print(json.dumps(out, indent=1))
    print("```")


if __name__ == "__main__":
    main(sys.argv[1:] or ["p64", "p128", "v256"])
