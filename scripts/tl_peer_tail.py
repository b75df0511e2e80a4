import ctypes as C, os, sys
import numpy as np
sys.path.insert(0, "/root/repo")
from paper_1905_01549_b200 import cgvk, problems as pb
P = pb.config_problem("p64"); nr = 8
lo = cgvk.partition_rows(P.A.n, nr, 4096)
mats = [cgvk.RankMatrix(P.A.n, lo, r, *cgvk.local_rows(P.A, lo, r)) for r in range(nr)]
comm = cgvk.Comm(nr)
lib = cgvk._lib; lib.cgvk_debug_timeline.argtypes = [C.c_void_p]
for v in ("pr", "hs", "gv", "cg"):
    g = cgvk.Group(comm, mats, cgvk.VariantConfig.make(cgvk.variant_from_name(v)), cgvk.Precond.JACOBI,
                   [P.b[lo[r]:lo[r+1]] for r in range(nr)], [P.x0[lo[r]:lo[r+1]] for r in range(nr)], p2p=True)
    s = g.solvers[0]; s.time_steps(20)
    buf = np.zeros((2, 1024, 8), np.uint64); lib.cgvk_debug_timeline(buf.ctypes.data)
    s.step(4); s.sync(); lib.cgvk_debug_timeline(buf.ctypes.data)
    for k in (0, 1):
        b = buf[k].astype(np.int64); live = b[:, 0] > 0
        if not live.any(): continue
        b = b[live]; t0 = b[:, 1].min()  # wait done
        last = np.argmax(b[:, 6])  # the CTA that published
        print(v, "kernel", k, "last CTA stamps rel. to wait-done (us): tiles done max", round((b[:,3].max()-t0)/1e3,2),
              "arrived", round((b[last,4]-t0)/1e3,2), "fold loads", round((b[last,7]-t0)/1e3,2),
              "tree done", round((b[last,5]-t0)/1e3,2), "published", round((b[last,6]-t0)/1e3,2))
    g.close()
