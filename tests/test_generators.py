"""Synthetic-input generators: RNG, structure, bitwise
symmetry, and the pinned sizes of the BASELINE configs (CPU only)."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1905_01549_b200 import problems as pb


def test_mt19937_64_known_answer():
    # C++ [rand.predef]: the 10000th output of a default-constructed
    # std::mt19937_64 (seed 5489) is 9981545732273789042.
    assert int(pb.mt19937_64(5489, 10000)[-1]) == 9981545732273789042


@pytest.mark.skipif(not O.reference_available(), reason="oracle/_ref not built")
def test_mt19937_64_matches_libstdcxx():
    for seed in (1, 7, 11, 2**63 + 5):
        assert np.array_equal(pb.mt19937_64(seed, 5000), O.ref_mt19937_64(seed, 5000))


def _check_csr(A: pb.CSR):
    n, rp, ci, va = A.n, A.row_ptr, A.col_idx, A.values
    assert rp[0] == 0 and rp[-1] == len(ci) == len(va)
    assert np.all(np.diff(rp) >= 0)
    assert ci.min() >= 0 and ci.max() < n
    rows = np.repeat(np.arange(n), np.diff(rp))
    # strictly increasing columns within rows
    same_row = rows[1:] == rows[:-1]
    assert np.all(ci[1:][same_row] > ci[:-1][same_row])
    # bit-symmetric: the transpose has identical pattern and value bits
    order = np.lexsort((rows, ci))
    t_rows, t_cols, t_vals = ci[order], rows[order], va[order]
    assert np.array_equal(t_rows, rows) and np.array_equal(t_cols, ci)
    assert np.array_equal(t_vals.view(np.int64), va.view(np.int64))


@pytest.mark.parametrize("N", [1, 2, 5, 16])
def test_poisson(N):
    A2, A3 = pb.poisson2d(N), pb.poisson3d(N)
    assert A2.nnz == 5 * N * N - 4 * N and A3.nnz == 7 * N**3 - 6 * N * N
    _check_csr(A2)
    _check_csr(A3)
    d = A3.values[A3.col_idx == np.repeat(np.arange(A3.n), np.diff(A3.row_ptr))]
    assert np.all(d == 6.0)


def test_varcoef_structure():
    A = pb.varcoef3d(12, seed=11, sigma=2.0)
    assert A.nnz == 7 * 12**3 - 6 * 144
    _check_csr(A)
    rows = np.repeat(np.arange(A.n), np.diff(A.row_ptr))
    off = A.col_idx != rows
    assert np.all(A.values[off] < 0)
    # diagonal = sum of face terms >= sum of |off-diagonals| (boundary faces add)
    absoff = np.bincount(rows[off], weights=-A.values[off], minlength=A.n)
    diag = A.values[~off]
    assert np.all(diag >= absoff * (1 - 1e-14))


def test_random_spd_structure():
    A = pb.random_spd(5000, 13, 400, 7)
    _check_csr(A)
    rows = np.repeat(np.arange(A.n), np.diff(A.row_ptr))
    assert np.all(np.abs(A.col_idx - rows) <= 400)
    # symmetric diagonal scaling of a diagonally dominant M-matrix: SPD; the
    # Jacobi-scaled matrix has unit diagonal and off-diagonal row sums < 1
    d = A.values[A.col_idx == rows]
    assert np.all(d > 0)


def test_baseline_sizes():
    # BASELINE.json configs; R4M nnz pinned by SURVEY E12 (113,033,524)
    assert pb.poisson2d(256).nnz == 326_656
    assert pb.poisson3d(64).nnz == 1_810_432
    A = pb.random_spd(1 << 22)
    assert A.n == 4_194_304 and A.nnz == 113_033_524


def test_xstar():
    x = pb.xstar(100000, 1)
    assert np.all((x > -1) & (x < 1)) and abs(x.mean()) < 0.02
    assert np.array_equal(x, pb.xstar(100000, 1))
    assert not np.array_equal(x, pb.xstar(100000, 2))


def test_rhs_in_reference_spmv_order():
    P = pb.config_problem("p2d")
    assert np.array_equal(P.b, O.spmv(P.A, P.x_star))
