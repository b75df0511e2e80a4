"""Extended-precision KATs of the device path — the reference's MPFR-based
tests (proj/tests/test_vector_ops.cpp, test_variants.cpp) restated with the
binary128 oracles of oracle/extprec.c (pinned in tests/test_extprec.py):

* the device dot (canonical tree) within the depth bound 64 eps sum|x_i y_i|
  of the exact dot, at sizes up to P128's n (the reference's own sequential
  dot is held to n eps |x||y|);
* every variant, on the reference test's 4x4 system, tracks CG carried in
  binary128 within 1e-12 for k = 1..4 (the reference checks HS);
* alpha_0 within one ulp of <r0,r0>/<p0,s0> evaluated exactly on the device
  state's own vectors (the reference: 'initialize alpha0 matches the exactly
  rounded ratio')."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1905_01549_b200 import cgvk, problems as pb
from paper_1905_01549_b200.cgvk import Precond, Variant, Vec

from extprec_cases import EPS, hilbert_shift_4
from helpers import ALL_VARIANTS

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [8, 4097, 262144, 2097152])
def test_device_dot_within_tree_bound_of_exact(n):
    rng = np.random.default_rng(n)
    x, y = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    # (the dot runs over a matrix's tiles: a diagonal matrix of size n)
    csr = pb.CSR(n, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int64), np.ones(n))
    A = cgvk.DeviceMatrix.from_csr(csr)
    got = A.dot(x, y)
    exact, scale = O.exact_dot(x, y), O.abs_dot(x, y)
    assert abs(got - exact) <= 64 * EPS * scale
    block, gmax, order = A.reduction_config()
    assert got == O.dot(x, y, ("tree", block, gmax, order))  # and it is the canonical tree


@pytest.mark.parametrize("variant", ALL_VARIANTS)
def test_variants_track_binary128_cg_on_the_4x4_system(variant):
    A, b, x0 = hilbert_shift_4()
    xs = O.high_prec_cg(A, b, x0, 4)
    D = cgvk.DeviceMatrix.from_csr(A)
    s = cgvk.initialize(cgvk.VariantConfig.make(variant), D, Precond.IDENTITY, b, x0)
    for k in range(4):
        s.step(1)
        s.sync()
        assert s.k == k + 1
        x = s.vector(Vec.X)
        assert np.linalg.norm(x - xs[k]) <= 1e-12 * np.linalg.norm(xs[k]), (variant.name, k)
    s.close()


@pytest.mark.parametrize("precond", [Precond.IDENTITY, Precond.JACOBI])
def test_alpha0_is_the_exactly_rounded_ratio(precond):
    P = pb.make_problem("p3", pb.poisson3d(20))
    rng = np.random.default_rng(7)
    b = rng.uniform(-1, 1, P.A.n)
    D = cgvk.DeviceMatrix.from_csr(P.A)
    s = cgvk.initialize(cgvk.VariantConfig.make(Variant.HS), D, precond, b, P.x0)
    r, p, sv = s.vector(Vec.R), s.vector(Vec.P), s.vector(Vec.S)
    rt = s.vector(Vec.R_TILDE) if precond == Precond.JACOBI else r
    exact = O.exact_ratio(rt, r, p, sv)
    alpha = s.scalars()["alpha"]
    assert abs(alpha - exact) <= np.spacing(abs(exact))
    s.close()
