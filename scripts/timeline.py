"""Phase timeline of one iteration's kernels (CGVK_TIMELINE=1 build):
per-CTA stamps 0 entry, 1 after griddepcontrol.wait, 2 first stage ready,
3 tiles done, 4 arrival counted, 5 fold done (last CTA), 6 finish done."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1905_01549_b200 import cgvk, problems as pb  # noqa: E402

args = [a for a in sys.argv[1:] if a != "--p2p"]
p2p = "--p2p" in sys.argv  # a one-rank peer-memory group instead of the single-GPU solver
cfg = args[0] if args else "p64"
P = pb.config_problem(cfg)
A = cgvk.DeviceMatrix.from_csr(P.A)
lib = cgvk._lib
lib.cgvk_debug_timeline.argtypes = [C.c_void_p]
if p2p:
    plane = {"p2d": 256, "p64": 4096, "p128": 16384, "v256": 65536}[cfg]
    nr = int(os.environ.get("TL_RANKS", "1"))  # in-process ranks (the stamps are the last rank's kernels)
    lo = cgvk.partition_rows(P.A.n, nr, plane)
    mats = [cgvk.RankMatrix(P.A.n, lo, r, *cgvk.local_rows(P.A, lo, r)) for r in range(nr)]
    comm = cgvk.Comm(nr)
for v in args[1:] or ["pr", "hs", "gv"]:
    cfgv = cgvk.VariantConfig.make(cgvk.variant_from_name(v))
    if p2p:
        g = cgvk.Group(comm, mats, cfgv, cgvk.Precond.JACOBI, [P.b[lo[r]:lo[r + 1]] for r in range(nr)],
                       [P.x0[lo[r]:lo[r + 1]] for r in range(nr)], p2p=True)
        s = g.solvers[0]
    else:
        s = cgvk.initialize(cfgv, A, cgvk.Precond.JACOBI, P.b, P.x0)
    s.time_steps(20)
    buf = np.zeros((2, 1024, 8), np.uint64)
    lib.cgvk_debug_timeline(buf.ctypes.data)  # read-and-clear
    s.step(int(os.environ.get("TL_STEPS", "1")))  # > 1: the last iteration's stamps (steady state)
    s.sync()
    assert lib.cgvk_debug_timeline(buf.ctypes.data) == 0
    print(f"== {cfg} {v}" + (" (one-rank peer-memory group)" if p2p else ""))
    t0 = None
    for k, name in ((0, "K1 update"), (1, "K2 spmv")):
        b = buf[k].astype(np.int64)
        live = b[:, 0] > 0
        b = b[live]
        if not len(b):  # one kernel per iteration (PrF): only the SpMV slot is stamped
            continue
        if t0 is None:
            t0 = b[:, 0].min()
        ent, wt, first, done, arr = (b[:, q] - t0 for q in range(5))
        fin = b[:, 6][b[:, 6] > 0] - t0 if (b[:, 6] > 0).any() else np.array([0])
        fold = b[:, 5][b[:, 5] > 0] - t0 if (b[:, 5] > 0).any() else np.array([0])
        loads = b[:, 7][b[:, 7] > 0] - t0 if (b[:, 7] > 0).any() else np.array([0])
        print(f"  {name}: CTAs {live.sum():4d} entry {ent.min()/1e3:6.2f}..{ent.max()/1e3:6.2f} us  "
              f"wait done {wt.min()/1e3:6.2f}..{wt.max()/1e3:6.2f}  first stage {first.min()/1e3:6.2f}..{first.max()/1e3:6.2f}  "
              f"tiles done {done.min()/1e3:6.2f}..{done.max()/1e3:6.2f}  arrived {arr.max()/1e3:6.2f}  "
              f"fold loads {loads.max()/1e3:6.2f} fold {fold.max()/1e3:6.2f}  finish {fin.max()/1e3:6.2f}")
        if os.environ.get("CGVK_CHAIN", "1") != "0" and (b[:, 5] > 0).all():
            pro = b[:, 5] - t0
            print(f"      chain prologue done {pro.min()/1e3:6.2f}..{pro.max()/1e3:6.2f}")
            if (b[:, 7] > 0).all() and (b[:, 4] > 0).all():
                c7, c4 = b[:, 7] - t0, b[:, 4] - t0
                print(f"      control block in smem {c7.min()/1e3:6.2f}..{c7.max()/1e3:6.2f}  "
                      f"partials folded {c4.min()/1e3:6.2f}..{c4.max()/1e3:6.2f}")
    (g if p2p else s).close()
