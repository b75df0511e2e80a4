"""Shape and structure edge cases through the C-ABI, bit-exact vs the oracle in
the device's reduction order: sizes around the 256-row tile boundary
(1, 255, 256, 257, ...), a tile whose CSR span exceeds the pipeline stage
(an arrow matrix: one dense row and column -> the stage's direct-load path),
a diagonal matrix, and seeded random SPD matrices of random size / density /
band for every variant and engine."""
import numpy as np
import pytest

from paper_1905_01549_b200 import cgvk, problems as pb
from paper_1905_01549_b200.cgvk import Precond, Variant

from helpers import ALL_VARIANTS, lockstep

pytestmark = pytest.mark.gpu


def arrow(n: int) -> pb.CSR:
    """SPD arrow: dense first row/column of -1/(n) plus a dominant diagonal."""
    rows, cols, vals = [], [], []
    for i in range(n):
        if i == 0:
            for j in range(n):
                rows.append(0), cols.append(j), vals.append(float(n) if j == 0 else -0.5)
        else:
            rows.append(i), cols.append(0), vals.append(-0.5)
            rows.append(i), cols.append(i), vals.append(2.0 + (i % 7) * 0.25)
    rows, cols, vals = np.array(rows), np.array(cols), np.array(vals)
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], vals[order]
    rp = np.zeros(n + 1, np.int64)
    np.add.at(rp, rows + 1, 1)
    return pb.CSR(n, np.cumsum(rp), cols.astype(np.int64), vals)


def diagonal(n: int) -> pb.CSR:
    return pb.CSR(n, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int64),
                  1.0 + np.arange(n) % 5)


@pytest.mark.parametrize("n", [1, 2, 255, 256, 257, 513, 4099])
@pytest.mark.parametrize("variant", [Variant.HS, Variant.CG_CG, Variant.PR, Variant.GV, Variant.PIPE_PR])
def test_tile_boundary_sizes(n, variant):
    P = pb.make_problem("rs", pb.random_spd(n, min(7, max(n - 1, 0)), max(n // 3, 1), 5))
    A = cgvk.DeviceMatrix.from_csr(P.A)
    lockstep(P.A, A, variant, Precond.JACOBI, P.b, P.x0, steps=10, check_vectors_every=5)


@pytest.mark.parametrize("variant", ALL_VARIANTS)
def test_dense_row_takes_the_direct_stage_path(variant):
    """Tile 0 holds a 20 000-entry row: more than a stage's CSR capacity, so
    the producer marks it direct and the consumers read A from global."""
    P = pb.make_problem("arrow", arrow(20000))
    A = cgvk.DeviceMatrix.from_csr(P.A)
    for precond in (Precond.IDENTITY, Precond.JACOBI):
        lockstep(P.A, A, variant, precond, P.b, P.x0, steps=8, check_vectors_every=4)


@pytest.mark.parametrize("variant", ALL_VARIANTS)
def test_diagonal_matrix(variant):
    P = pb.make_problem("diag", diagonal(3000))
    A = cgvk.DeviceMatrix.from_csr(P.A)
    lockstep(P.A, A, variant, Precond.IDENTITY, P.b, P.x0, steps=6, check_vectors_every=1)


@pytest.mark.parametrize("seed", range(8))
def test_random_structures(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(300, 30000))
    per_row = int(rng.integers(1, 20))
    band = int(rng.integers(1, max(2, min(n // 2, 6000))))
    P = pb.make_problem("fz", pb.random_spd(n, per_row, band, 100 + seed))
    engine = [None, "csr", "band"][seed % 3]
    A = cgvk.DeviceMatrix.from_csr(P.A, engine=engine)
    variant = ALL_VARIANTS[seed % len(ALL_VARIANTS)]
    precond = [Precond.IDENTITY, Precond.JACOBI][seed % 2]
    lockstep(P.A, A, variant, precond, P.b, P.x0, steps=12, check_vectors_every=4)
