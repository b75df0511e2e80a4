import time, sys
sys.path.insert(0, '.')
from paper_1905_01549_b200 import cgvk, problems as pb
from paper_1905_01549_b200.cgvk import Precond, Variant, VariantConfig
P = pb.config_problem("p128")
A = P.A
lo = cgvk.partition_rows(A.n, 2, 128*128)
comm = cgvk.Comm(2)
for rep in range(2):
    t = time.perf_counter()
    parts = [cgvk.local_rows(A, lo, r) for r in range(2)]
    t1 = time.perf_counter()
    mats = [cgvk.RankMatrix(A.n, lo, r, *parts[r]) for r in range(2)]
    t2 = time.perf_counter()
    gs = []
    for v in (Variant.HS, Variant.GV):
        for p2p in (True, False):
            t3 = time.perf_counter()
            g = cgvk.Group(comm, mats, VariantConfig.make(v), Precond.JACOBI, [P.b[lo[r]:lo[r+1]] for r in range(2)], [P.x0[lo[r]:lo[r+1]] for r in range(2)], p2p=p2p)
            print(v.name, p2p, "group %.1f ms" % (1e3*(time.perf_counter()-t3)), file=sys.stderr)
            gs.append(g)
    print("local_rows %.1f ms, rank matrices %.1f ms" % (1e3*(t1-t), 1e3*(t2-t1)), file=sys.stderr)
    for g in gs: g.close()
    for m in mats: m.close()
