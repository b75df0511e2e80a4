import os, sys, time
sys.path.insert(0, ".")
os.environ["CGVK_P2P_DELAY_NS"] = str(int(2.1e9))
from paper_1905_01549_b200 import cgvk, problems as pb
from paper_1905_01549_b200.cgvk import Precond, Variant
P = pb.make_problem("p", pb.poisson3d(12))
A = P.A
lo = cgvk.partition_rows(A.n, 1, 144)
mats = [cgvk.RankMatrix(A.n, lo, 0, *cgvk.local_rows(A, lo, 0))]
comm = cgvk.Comm(1)
t = time.time()
g = cgvk.Group(comm, mats, cgvk.VariantConfig.make(Variant.HS), Precond.JACOBI, [P.b], [P.x0], p2p=True)
print("create", time.time() - t, g.transport, flush=True)
t = time.time()
g.step(1)
print("step enq", time.time() - t, flush=True)
t = time.time()
try:
    g.sync()
    print("sync ok", time.time() - t, g.solvers[0].k, flush=True)
except Exception as e:
    print("sync raised", type(e).__name__, e, time.time() - t, flush=True)
