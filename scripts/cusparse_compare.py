"""Library comparator for the SpMV ("cuSPARSE CSR SpMV is a
useful sanity comparator, not a target"): cuSPARSE's fp64 CSR SpMV (through
torch.sparse CSR, int32 and int64 indices) on the BASELINE matrices, next to
this library's standalone SpMV (cgvk_spmv, the generic kernel) and its fused
SpMV kernels (K2 of each variant: the SpMV plus that variant's vector updates
and dot products), all CUDA-event timed, with the algorithmic bytes of one
SpMV (12 B/nnz + 4(n+1) + 16 n: A, x read once, y written) per launch.

usage: python scripts/cusparse_compare.py [configs...] > profiles/r02/cusparse.md
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1905_01549_b200 import cgvk, problems as pb  # noqa: E402

PEAK = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6550.0


def ev_time(fn, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps  # ms


def main(configs):
    out = {}
    print("# SpMV: cuSPARSE vs this library (round 2)\n")
    print(__doc__.split("usage:")[0].strip().replace("\n", " ") + "\n")
    print("| config | bytes / SpMV (MB) | cuSPARSE int32 us (GB/s) | cuSPARSE int64 us (GB/s) | "
          "cgvk_spmv us (GB/s) | fused K2 us per variant (SpMV + its vector work) |")
    print("|---|---:|---:|---:|---:|---|")
    for cfg in configs:
        P = pb.config_problem(cfg)
        A = P.A
        n, nnz = A.n, A.nnz
        mb = (12 * nnz + 4 * (n + 1) + 16 * n) / 1e6
        x = torch.from_numpy(P.x_star).cuda()
        res = {}
        for idx in (torch.int32, torch.int64):
            T = torch.sparse_csr_tensor(torch.from_numpy(A.row_ptr).to(idx), torch.from_numpy(A.col_idx).to(idx),
                                        torch.from_numpy(A.values), size=(n, n)).cuda()
            ms = ev_time(lambda: torch.mv(T, x))
            y = torch.mv(T, x).cpu().numpy()
            res[str(idx)] = (1e3 * ms, mb / ms)
            del T
        D = cgvk.DeviceMatrix.from_csr(A)
        ours_ms = D.time_ops(50)["spmv"]
        ref = D.spmv(P.x_star)
        same = bool(np.array_equal(ref.view(np.int64), A.spmv(P.x_star).view(np.int64)))
        fused = {}
        for v in ("hs", "cg", "pr", "gv", "pipe-pr"):
            s = cgvk.initialize(cgvk.VariantConfig.make(cgvk.variant_from_name(v)), D, cgvk.Precond.JACOBI,
                                P.b, P.x0)
            s.time_steps(5)
            a, b2, it = s.profile(50)
            fused[v] = 1e3 * b2 / max(it, 1)
            s.close()
        D.close()
        cus_err = float(np.max(np.abs(y - ref)) / np.max(np.abs(ref)))
        out[cfg] = {"mb": mb, "cusparse": res, "cgvk_spmv_us": 1e3 * ours_ms, "fused_k2_us": fused,
                    "cgvk_bits_equal_reference_order": same, "cusparse_max_rel_diff": cus_err}
        c32, c64 = res["torch.int32"], res["torch.int64"]
        print(f"| {cfg} | {mb:.1f} | {c32[0]:.1f} ({c32[1]:.0f}) | {c64[0]:.1f} ({c64[1]:.0f}) | "
              f"{1e3 * ours_ms:.1f} ({mb / ours_ms:.0f}) | "
              + ", ".join(f"{k} {u:.1f}" for k, u in fused.items()) + " |")
    print("\ncgvk's SpMV is bit-identical to the reference's row order (`cgvk_bits_equal_reference_order`); "
          "cuSPARSE's is not bound to it (`cusparse_max_rel_diff`).\n")
    print("```json")
    print(json.dumps(out, indent=1))
    print("```")


if __name__ == "__main__":
    main(sys.argv[1:] or ["p64", "p128", "v256", "r4m"])
