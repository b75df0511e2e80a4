"""Print the launch configuration (occupancy, grid, smem, ring depth) of every
pipeline kernel of each variant on a BASELINE config (CGVK_DEBUG=1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["CGVK_DEBUG"] = "1"
from paper_1905_01549_b200 import cgvk, problems as pb
P = pb.config_problem(sys.argv[1] if len(sys.argv) > 1 else "p128")
A = cgvk.DeviceMatrix.from_csr(P.A)
for v in ["hs", "cg", "pr", "gv", "pipe-pr"]:
    print("==", v, file=sys.stderr, flush=True)
    s = cgvk.initialize(cgvk.VariantConfig.make(cgvk.variant_from_name(v)), A, cgvk.Precond.JACOBI, P.b, P.x0)
    s.close()
