"""Cost-model calibration on one B200.

For each config: measure the model's parameters on the device
(paper_1905_01549_b200.cost_model.calibrate: SpMV, one-pass block SpMV, one
global reduction), the fused solver's measured time per iteration for every
variant (CUDA events, graph-replayed), and print the model's prediction next
to it. Then a strong-scaling scenario for 1/2/4/8 GPUs: t_mv, t_2mv divided
by P (measured 1-GPU values), c_mv = halo bytes over NVLink + a latency, c_gr =
the 1-GPU reduction + an allreduce latency; the two latencies are ASSUMED
(one GPU per call here), so the crossovers are shown for a range of them.

usage: python scripts/cost_model.py [configs...] > profiles/r01/cost_model.md
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1905_01549_b200 import cgvk, problems as pb  # noqa: E402
from paper_1905_01549_b200.cgvk import Precond, Variant, VariantConfig  # noqa: E402
from paper_1905_01549_b200.cost_model import (CostParams, ScalingScenario, calibrate,  # noqa: E402
                                              crossover_nodes, iteration_time)

VARIANTS = [Variant.HS, Variant.CG_CG, Variant.M, Variant.PR, Variant.GV, Variant.PIPE_PR]
PLANE = {"p64": 64 * 64, "p128": 128 * 128, "v256": 256 * 256, "r4m": 4096, "p2d": 256}
NVLINK_GBS = 900.0  # per direction, per GPU (NVLink 5 / NVSwitch)


def measured_us(A, P, v, iters=100):
    s = cgvk.initialize(VariantConfig.make(v), A, Precond.JACOBI, P.b, P.x0)
    s.time_steps(5)
    ms, it = s.time_steps(iters)
    s.close()
    return 1e3 * ms / max(it, 1)


def main(configs):
    out = {}
    print("# Cost-model calibration (src/cost_model.cpp) on one B200\n")
    print("Parameters measured with `cgvk_time_ops` (CUDA events, generic L1 kernels); "
          "iteration times are the fused solver's (graph-replayed, Jacobi). "
          "The model ignores vector updates and local dots, which on one GPU are "
          "as HBM-bound as the SpMV itself, so it under-predicts; its *ordering* "
          "is what the strong-scaling scenario below uses. t_mv / t_2mv are the "
          "generic CSR kernels (x through L1), so on R4M they exceed the band "
          "engine's fused SpMV.\n")
    for cfg in configs:
        P = pb.config_problem(cfg)
        A = cgvk.DeviceMatrix.from_csr(P.A)
        p, ms = calibrate(A)
        rows = []
        for v in VARIANTS:
            pred = iteration_time(v, p) * 1e6
            meas = measured_us(A, P, v)
            rows.append((v.name, pred, meas))
        out[cfg] = {"ms": ms, "params_us": {k: 1e6 * getattr(p, k) for k in ("c_gr", "t_mv", "c_mv", "t_2mv")},
                    "variants": {r[0]: {"model_us": r[1], "measured_us": r[2]} for r in rows}}
        print(f"## {cfg} (n = {P.A.n:,}, nnz = {P.A.nnz:,}; engine {A.engine()[0]})\n")
        print(f"c_gr = {1e6 * p.c_gr:.1f} us (one global reduction), t_mv = {1e6 * p.t_mv:.1f} us, "
              f"t_2mv = {1e6 * p.t_2mv:.1f} us, c_mv = 0 (one GPU); vector copy {1e3 * ms['copy']:.1f} us\n")
        print("| variant | model us/iter | measured us/iter (fused kernels) | measured / model |")
        print("|---|---:|---:|---:|")
        for name, pred, meas in rows:
            print(f"| {name} | {pred:.1f} | {meas:.1f} | {meas / pred:.2f} |")
        print()
        # strong-scaling scenario over one NVSwitch box
        halo = 8.0 * PLANE.get(cfg, 4096)  # bytes per neighbour per vector
        print("Strong-scaling scenario (assumed allreduce latency L_ar and halo latency L_h; "
              "t_mv, t_2mv / P from the 1-GPU measurement):\n")
        print("| L_ar (us) | L_h (us) | HS us/iter @1,2,4,8 | GV | pipe-PR | GV beats HS from | pipe-PR beats PR from |")
        print("|---:|---:|---|---|---|---:|---:|")
        for l_ar, l_h in ((5.0, 3.0), (10.0, 5.0), (20.0, 8.0)):
            nodes = [1, 2, 4, 8]
            params = []
            for n in nodes:
                c_gr = p.c_gr + (l_ar * 1e-6 if n > 1 else 0.0)
                c_mv = (l_h * 1e-6 + halo / (NVLINK_GBS * 1e9)) if n > 1 else 0.0
                params.append(CostParams(c_gr, p.t_mv / n, c_mv, p.t_2mv / n))
            sc = ScalingScenario(nodes, params)

            def series(v):
                return ", ".join(f"{1e6 * iteration_time(v, q):.0f}" for q in params)

            cx1 = crossover_nodes(Variant.GV, Variant.HS, sc)
            cx2 = crossover_nodes(Variant.PIPE_PR, Variant.PR, sc)
            print(f"| {l_ar:.0f} | {l_h:.0f} | {series(Variant.HS)} | {series(Variant.GV)} | "
                  f"{series(Variant.PIPE_PR)} | {cx1} | {cx2} |")
        print()
        A.close()
    print("```json")
    print(json.dumps(out, indent=1))
    print("```")


if __name__ == "__main__":
    main(sys.argv[1:] or ["p64", "p128", "r4m"])
