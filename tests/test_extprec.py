"""The binary128 oracles (oracle/extprec.c: exact dot, exact ratio, CG
carried in binary128) pinned on the CPU — against exact rational arithmetic
and against the reference's own solver — so the GPU extended-precision KATs
(tests/test_gpu_extprec.py) rest on a checked oracle."""
from fractions import Fraction

import numpy as np
import pytest

from oracle import oracle as O
from paper_1905_01549_b200 import problems as pb

from extprec_cases import EPS, hilbert_shift_4


@pytest.mark.parametrize("n,seed", [(8, 2024), (1000, 3), (4097, 5)])
def test_exact_dot_is_exactly_rounded(n, seed):
    rng = np.random.default_rng(seed)
    x, y = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    exact = sum(Fraction(float(a)) * Fraction(float(b)) for a, b in zip(x, y))
    assert O.exact_dot(x, y) == float(exact)
    num = sum(Fraction(float(a)) * Fraction(float(a)) for a in x)
    den = sum(Fraction(float(b)) * Fraction(float(b)) for b in y)
    assert O.exact_ratio(x, x, y, y) == float(num / den)


@pytest.mark.parametrize("n", [8, 1000, 65536])
def test_sequential_and_tree_dots_within_their_error_bounds(n):
    """The reference's dot (sequential) within its n*eps*|x||y| model bound
    (proj/tests/test_vector_ops.cpp), and the device's canonical tree —
    restated by the oracle — within the much tighter depth bound."""
    rng = np.random.default_rng(n)
    x, y = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    exact, scale = O.exact_dot(x, y), O.abs_dot(x, y)
    seq = O.dot(x, y, "seq")
    assert abs(seq - exact) <= n * EPS * np.linalg.norm(x) * np.linalg.norm(y)
    tree = O.dot(x, y, ("tree", 256, 444, 0))
    assert abs(tree - exact) <= 64 * EPS * scale


def test_high_prec_cg_matches_the_reference_hs_on_the_4x4_system():
    """The binary128 CG and the reference's own HS (oracle/_ref) agree within
    the reference test's 1e-12 for k = 1..4 (proj/tests/test_variants.cpp)."""
    A, b, x0 = hilbert_shift_4()
    xs = O.high_prec_cg(A, b, x0, 4)
    assert xs.shape == (4, 4)
    runs = [O.Restatement(A, 0, 0, b, x0)]
    if O.reference_available():
        runs.append(O.Reference(A, 0, 0, b, x0))
    for run in runs:
        for k in range(4):
            run.step()
            x = run.vector(0)
            assert np.linalg.norm(x - xs[k]) <= 1e-12 * np.linalg.norm(xs[k])


def test_high_prec_cg_converges_to_the_solution():
    P = pb.make_problem("p2", pb.poisson2d(12))
    d = 1.0 / np.array([P.A.values[(P.A.col_idx == i) & (np.repeat(np.arange(P.A.n), np.diff(P.A.row_ptr)) == i)][0]
                        for i in range(P.A.n)])
    xs = O.high_prec_cg(P.A, P.b, P.x0, 200, inv_diag=d)
    assert np.linalg.norm(xs[-1] - P.x_star) <= 1e-12 * np.linalg.norm(P.x_star)
