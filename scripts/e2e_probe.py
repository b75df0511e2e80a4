"""Break the e2e sweep (bench.py) into matrix upload / solver init / steps."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1905_01549_b200 import cgvk, problems as pb
from paper_1905_01549_b200.cgvk import Precond, VariantConfig, variant_from_name
P = pb.config_problem(sys.argv[1] if len(sys.argv) > 1 else "p128")
arrs = [P.A.row_ptr.copy(), P.A.col_idx.copy(), P.A.values.copy(), P.b.copy(), P.x0.copy()]
for a in arrs:
    cgvk.host_register(a)
for rep in range(3):
    t0 = time.perf_counter()
    A = cgvk.DeviceMatrix(P.A.n, *arrs[:3])
    t1 = time.perf_counter()
    ss = []
    tinit = tstep = 0
    for v in ["hs", "cg", "m", "pr", "gv", "pipe-pr"]:
        a = time.perf_counter()
        s = cgvk.initialize(VariantConfig.make(variant_from_name(v)), A, Precond.JACOBI, arrs[3], arrs[4])
        b = time.perf_counter()
        s.step(200); s.sync(); x = s.x
        c = time.perf_counter()
        tinit += b - a; tstep += c - b
        ss.append(s)
    for s in ss: s.close()
    A.close()
    t2 = time.perf_counter()
    print(f"matrix {1e3*(t1-t0):.1f} ms  init {1e3*tinit:.1f} ms  steps+x {1e3*tstep:.1f} ms  total {1e3*(t2-t0):.1f} ms", flush=True)
