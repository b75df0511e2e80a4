"""Per-variant time per iteration of one rank's solve three ways: the
single-GPU solver, a one-rank group over the copy exchange, a one-rank group
over peer memory — the cost of the rank machinery itself (no neighbour)."""
import sys

sys.path.insert(0, ".")
from paper_1905_01549_b200 import cgvk, problems as pb  # noqa: E402
from paper_1905_01549_b200.cgvk import Precond, Variant, VariantConfig  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "p128"
P = pb.config_problem(cfg)
A = P.A
plane = {"p64": 4096, "p128": 16384, "v256": 65536}[cfg]
D = cgvk.DeviceMatrix.from_csr(A)
lo = cgvk.partition_rows(A.n, 1, plane)
mats = [cgvk.RankMatrix(A.n, lo, 0, *cgvk.local_rows(A, lo, 0))]
comm = cgvk.Comm(1)
for v in (Variant.HS, Variant.CG_CG, Variant.PR, Variant.GV, Variant.PIPE_PR):
    row = []
    s = cgvk.initialize(VariantConfig.make(v), D, Precond.JACOBI, P.b, P.x0)
    s.time_steps(5)
    ms, it = s.time_steps(200)
    row.append(1e3 * ms / it)
    s.close()
    for p2p in (False, True):
        g = cgvk.Group(comm, mats, VariantConfig.make(v), Precond.JACOBI, [P.b], [P.x0], p2p=p2p)
        s = g.solvers[0]
        s.time_steps(5)
        ms, it = s.time_steps(200)
        row.append(1e3 * ms / it)
        g.close()
    print(f"{v.name:8s} single {row[0]:6.1f}  group-copy {row[1]:6.1f}  group-p2p {row[2]:6.1f} us/iter", flush=True)
