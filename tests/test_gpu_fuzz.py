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


@pytest.mark.parametrize("band,want", [(19 * 256 - 255, "band"), (21 * 256, "csr")])
def test_band_window_limit(band, want):
    """Half-width H = 19 tiles is the largest window the band engine keeps;
    a wider band stays on CSR. Both bit-exact."""
    P = pb.make_problem("bw", pb.random_spd(40000, 13, band, 17))
    A = cgvk.DeviceMatrix.from_csr(P.A)
    assert A.engine()[0] == want
    for v in (Variant.HS, Variant.PIPE_PR):
        lockstep(P.A, A, v, Precond.JACOBI, P.b, P.x0, steps=6, check_vectors_every=6)


@pytest.mark.parametrize("seed", range(6))
def test_random_l1_operators(seed):
    from oracle import oracle as O
    from helpers import same_bits, tree_dot
    rng = np.random.default_rng(50 + seed)
    n = int(rng.integers(1, 20000))
    P = pb.make_problem("l1", pb.random_spd(n, int(rng.integers(0, 16)), int(rng.integers(1, max(2, n))),
                                            200 + seed))
    A = cgvk.DeviceMatrix.from_csr(P.A, engine=[None, "band", "csr"][seed % 3])
    x1, x2 = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    assert same_bits(A.spmv(x1), O.spmv(P.A, x1))
    y1, y2 = A.block_spmv(x1, x2)
    assert same_bits(y1, O.spmv(P.A, x1)) and same_bits(y2, O.spmv(P.A, x2))
    assert same_bits(A.jacobi(), O.jacobi(P.A))
    assert same_bits(np.float64(A.dot(x1, x2)), np.float64(O.dot(x1, x2, tree_dot(A))))


@pytest.mark.parametrize("seed", range(6))
def test_random_partitioned_solves(seed):
    """Row-partitioned (local transport) solves of random structures, P = 2..5
    ranks, bit-exact vs the partitioned oracle."""
    from oracle import oracle as O
    from test_gpu_group import compare
    rng = np.random.default_rng(70 + seed)
    n = int(rng.integers(2000, 40000))
    nranks = int(rng.integers(2, 6))
    P = pb.make_problem("pp", pb.random_spd(n, int(rng.integers(2, 14)), int(rng.integers(8, n // (2 * nranks))),
                                            300 + seed))
    lo = cgvk.partition_rows(n, nranks, 1)
    mats = [cgvk.RankMatrix(n, lo, r, *cgvk.local_rows(P.A, lo, r)) for r in range(nranks)]
    comm = cgvk.Comm(nranks)
    variant = ALL_VARIANTS[seed % len(ALL_VARIANTS)]
    g = cgvk.Group(comm, mats, cgvk.VariantConfig.make(variant), Precond.JACOBI,
                   [P.b[lo[r]:lo[r + 1]] for r in range(nranks)], [P.x0[lo[r]:lo[r + 1]] for r in range(nranks)])
    block, gmax, order = mats[0].reduction_config()
    o = O.Restatement(P.A, int(variant), 1, P.b, P.x0, dot=("part", block, gmax, lo, order))
    for k in range(8):
        g.step(1)
        g.sync()
        if o.state()["state"] == 0:
            o.step()
    compare(g, o, f"fuzz-part seed {seed} P{nranks} {variant.name}")
    g.close()
    comm.close()


@pytest.mark.parametrize("engine", [None, "band"])
@pytest.mark.parametrize("variant", ALL_VARIANTS)
def test_chained_graph_steps_match_the_oracle(variant, engine):
    """step(n) replays graphs of chained iterations (each K1 after the first
    runs the previous K2's scalar tail, the graph's tail kernel the last
    one): 8 + 8 + 3 iterations in one call, then the oracle's 19 steps."""
    from oracle import oracle as O
    from helpers import compare_states, compare_vectors, gpu_state, gpu_vectors, oracle_vectors, tree_dot
    P = pb.make_problem("ch", pb.random_spd(20000, 13, 3000, 21))
    A = cgvk.DeviceMatrix.from_csr(P.A, engine=engine)
    for precond in (Precond.IDENTITY, Precond.JACOBI):
        s = cgvk.initialize(cgvk.VariantConfig.make(variant), A, precond, P.b, P.x0)
        o = O.Restatement(P.A, int(variant), int(precond), P.b, P.x0, dot=tree_dot(A))
        s.step(19)
        s.sync()
        for _ in range(19):
            if o.state()["state"] != 0:
                break
            o.step()
        compare_states(gpu_state(s), o.state(), f"{variant.name} chained x19")
        compare_vectors(gpu_vectors(s), oracle_vectors(o), f"{variant.name} chained x19")
        s.close()


def test_last_cta_schedule_still_bit_exact():
    """CGVK_CHAIN=0 captures the last-CTA schedule (A/B): same bits."""
    import os
    import subprocess
    import sys
    code = ("import sys; sys.path[:0] = ['tests', '.']\n"
            "from test_gpu_fuzz import test_chained_graph_steps_match_the_oracle as t\n"
            "from helpers import ALL_VARIANTS\n"
            "for v in ALL_VARIANTS:\n"
            "    t(v, None)\n"
            "print('ok')\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=dict(os.environ, CGVK_CHAIN="0"),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-2000:]
