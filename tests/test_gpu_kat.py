"""Table-3 KAT sweep on the GPU path: the nine bundled
Matrix-Market fixtures (parsed by the reference parser into
tests/golden/mtx), x* = 1/sqrt(n), x0 = 0, stop at a relative A-norm error
< 1e-5 (the protocol of proj/tests/test_matrices.cpp:27-46). The GPU solve
must reproduce the reference's iteration counts (tests/golden/table3.json)
within the reference tests' own windows, and the paper's published numbers
(PAPER.md:819-879)."""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_1905_01549_b200 import cgvk, problems as pb
from paper_1905_01549_b200.cgvk import Precond, Variant

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

VIDS = {"hs": Variant.HS, "cg": Variant.CG_CG, "m": Variant.M, "pr": Variant.PR, "gv": Variant.GV,
        "pipe-pr-m": Variant.PIPE_PR_M, "pipe-pr": Variant.PIPE_PR}

with open(os.path.join(GOLDEN, "table3.json")) as f:
    TABLE3 = json.load(f)

# keep the sweep short: skip the 30k-iteration nos2 and the long-budget runs
KEYS = [k for k, v in sorted(TABLE3["runs"].items())
        if not k.startswith("nos2/") and 0 <= v["iters_to_1e5"] <= 1500]


def load(name):
    d = np.load(os.path.join(GOLDEN, "mtx", name + ".npz"))
    return pb.CSR(int(d["n"]), d["row_ptr"], d["col_idx"], d["values"])


_mats = {}


def gpu_iters_to_1e5(name, v, prec, budget):
    A = load(name)
    if name not in _mats:
        _mats.clear()
        _mats[name] = cgvk.DeviceMatrix.from_csr(A)
    D = _mats[name]
    xs = np.full(A.n, 1.0 / np.sqrt(A.n))
    b = A.spmv(xs)
    s = cgvk.initialize(cgvk.VariantConfig.make(v), D, prec, b, np.zeros(A.n))

    def rel_err():
        e = xs - s.x
        q = O.dot(e, O.spmv(A, e), "seq")  # a_norm of src/sparse_matrix.cpp:169-178
        return np.sqrt(max(q, 0.0))

    e0 = rel_err()
    for _ in range(budget):
        if not s.status.running():
            return -1
        cgvk.step(s)
        if rel_err() / e0 < 1e-5:
            return s.k
    return -1


# On the ill-conditioned fixtures (bcsstk03, 494_bus, 1138_bus and nos7
# unpreconditioned) the iteration count itself depends on the summation order
# of the dots (finite-precision convergence delay, §3): the
# tree-order CPU oracle differs from the sequential reference by up to 7.1 %
# (bcsstk03 GV: 605 vs 565). The GPU must equal the tree-order oracle
# exactly and the reference within that measured floor.
REORDER_FLOOR = 0.08


@pytest.mark.parametrize("key", KEYS)
def test_table3_on_gpu(key):
    name, prec, v = key.split("/")
    gold = TABLE3["runs"][key]
    pc = Precond.JACOBI if prec == "jacobi" else Precond.IDENTITY
    got = gpu_iters_to_1e5(name, VIDS[v], pc, int(gold["iters_to_1e5"] * 1.2) + 50)
    A = load(name)
    xs = np.full(A.n, 1.0 / np.sqrt(A.n))
    block, gmax, order = _mats[name].reduction_config()
    o = O.Restatement(A, int(VIDS[v]), int(pc), A.spmv(xs), np.zeros(A.n), dot=("tree", block, gmax, order))
    tree = o.anorm_run(xs, gold["budget"], 1e-5)["iters_to_1e5"]
    assert got == tree, (key, got, tree)
    ref = gold["iters_to_1e5"]
    assert abs(got - ref) <= max(3, REORDER_FLOOR * ref), (key, got, ref)


def test_published_table3_rows_on_gpu():
    """PAPER.md:832-870 via the GPU path: nos4 72, nos7+Jacobi 67, bcsstm22 43, bcsstm21 3."""
    assert gpu_iters_to_1e5("bcsstm21", Variant.HS, Precond.IDENTITY, 50) == 3
    assert abs(gpu_iters_to_1e5("bcsstm22", Variant.PIPE_PR, Precond.IDENTITY, 300) - 43) <= 1
    for v in Variant:
        assert abs(gpu_iters_to_1e5("nos4", v, Precond.IDENTITY, 400) - 72) <= 2
        assert abs(gpu_iters_to_1e5("nos7", v, Precond.JACOBI, 400) - 67) <= 3
