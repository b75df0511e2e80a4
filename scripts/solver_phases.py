"""Host-side cost of cgvk_solver_create per variant (CGVK_DEBUG=2 phase timers)."""
import sys
import time

sys.path.insert(0, ".")
from paper_1905_01549_b200 import cgvk, problems as pb  # noqa: E402
from paper_1905_01549_b200.cgvk import Precond, Variant, VariantConfig  # noqa: E402

P = pb.config_problem(sys.argv[1] if len(sys.argv) > 1 else "p128")
A = cgvk.DeviceMatrix.from_csr(P.A)
for rep in range(2):
    for v in (Variant.HS, Variant.GV, Variant.PIPE_PR):
        t = time.perf_counter()
        s = cgvk.initialize(VariantConfig.make(v), A, Precond.JACOBI, P.b, P.x0)
        t1 = time.perf_counter()
        s.step(20)
        s.sync()
        t2 = time.perf_counter()
        print(f"{v.name}: create {1e3 * (t1 - t):.2f} ms, step(20)+sync {1e3 * (t2 - t1):.2f} ms", file=sys.stderr)
        s.close()
