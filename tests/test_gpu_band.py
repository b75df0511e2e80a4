"""Band engine (SELL-C-sigma + shared-memory x window, cgvk_band.cuh) vs the
oracle, through the C-ABI.

The band engine runs the SpMV kernel (K2) of every variant for narrow-band,
long-row matrices (BASELINE config R4M). Its rows are permuted inside each
256-row tile and its columns stored as 16-bit window offsets, but every row
sum keeps the reference's CSR order and the dot contributions are folded in
the canonical tile-contiguous order (reduction_config() reports order 1), so
the whole trajectory must be bit-identical to the tree-order restatement.
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1905_01549_b200 import cgvk, problems as pb
from paper_1905_01549_b200.cgvk import Precond, Variant

from helpers import ALL_VARIANTS, lockstep, same_bits

pytestmark = pytest.mark.gpu


def _problems():
    return {
        "randspd_3000": pb.make_problem("rs", pb.random_spd(3000, 13, 300, 7)),
        "randspd_20000_b4096": pb.make_problem("rs2", pb.random_spd(20000, 13, 4096, 9)),
        "poisson2d_33": pb.make_problem("p2", pb.poisson2d(33)),        # ragged last tile, H = 1
        "poisson3d_12": pb.make_problem("p3", pb.poisson3d(12)),
        "tiny_100": pb.make_problem("t", pb.random_spd(100, 5, 50, 3)),  # one partial tile
    }


PROBLEMS = _problems()


@pytest.fixture(scope="module")
def bandmats():
    return {k: cgvk.DeviceMatrix.from_csr(p.A, engine="band") for k, p in PROBLEMS.items()}


def test_engine_selection():
    rs = cgvk.DeviceMatrix.from_csr(PROBLEMS["randspd_20000_b4096"].A)
    assert rs.engine() == ("band", 16)
    assert rs.reduction_config()[2] == 1
    p3 = cgvk.DeviceMatrix.from_csr(PROBLEMS["poisson3d_12"].A)
    assert p3.engine() == ("csr", 0)  # short rows: L1 gathers
    assert cgvk.DeviceMatrix.from_csr(PROBLEMS["randspd_3000"].A, engine="csr").engine()[0] == "csr"
    # a band wider than the window budget stays on CSR even when asked
    wide = cgvk.DeviceMatrix.from_csr(pb.random_spd(30000, 13, 12000, 5), engine="band")
    assert wide.engine() == ("csr", 0)


@pytest.mark.parametrize("name", list(PROBLEMS))
def test_band_engine_applies(name, bandmats):
    assert bandmats[name].engine()[0] == "band"


@pytest.mark.parametrize("precond", [Precond.IDENTITY, Precond.JACOBI])
@pytest.mark.parametrize("variant", ALL_VARIANTS)
@pytest.mark.parametrize("name", list(PROBLEMS))
def test_band_trajectory_bit_exact(name, variant, precond, bandmats):
    P = PROBLEMS[name]
    lockstep(P.A, bandmats[name], variant, precond, P.b, P.x0, steps=20, check_vectors_every=5)


@pytest.mark.parametrize("cfg", [{"recompute_w": 0}, {"unsimplified_mu": 1}, {"track_delta": 1}],
                         ids=["no_recompute_w", "unsimplified_mu", "track_delta"])
def test_band_ablations_bit_exact(cfg, bandmats):
    P = PROBLEMS["randspd_20000_b4096"]
    key = next(iter(cfg))
    variants = {"recompute_w": [Variant.PIPE_PR, Variant.PIPE_PR_M],
                "unsimplified_mu": [Variant.CG_CG, Variant.GV],
                "track_delta": [Variant.PR, Variant.PIPE_PR]}[key]
    for v in variants:
        lockstep(P.A, bandmats["randspd_20000_b4096"], v, Precond.JACOBI, P.b, P.x0, steps=12,
                 cfg_kwargs=cfg, check_vectors_every=4)


def test_band_many_tiles_per_virtual_cta():
    """n = 600k: 2344 tiles > the 888 virtual CTAs (6 x 148), so CTAs walk multi-tile
    runs and the window ring wraps many times."""
    P = pb.make_problem("rs_big", pb.random_spd(600_000, 13, 4096, 11))
    A = cgvk.DeviceMatrix.from_csr(P.A)
    assert A.engine() == ("band", 16)
    for v in (Variant.HS, Variant.PR, Variant.PIPE_PR):
        lockstep(P.A, A, v, Precond.JACOBI, P.b, P.x0, steps=6, check_vectors_every=6)


def test_band_vs_csr_engine_histories():
    """Both engines on one matrix: reduction orders differ (tiles strided vs
    contiguous), residual histories agree to 1e-10 relative over 50 steps."""
    P = PROBLEMS["randspd_20000_b4096"]
    Ab = cgvk.DeviceMatrix.from_csr(P.A, engine="band")
    Ac = cgvk.DeviceMatrix.from_csr(P.A, engine="csr")
    for v in ALL_VARIANTS:
        h = []
        for A in (Ab, Ac):
            s = cgvk.initialize(cgvk.VariantConfig.make(v), A, Precond.JACOBI, P.b, P.x0)
            s.step(50)
            s.sync()
            h.append(np.sqrt(s.history()))
        n = min(len(h[0]), len(h[1]))
        assert n >= 40
        rel = np.abs(h[0][:n] - h[1][:n]) / np.maximum(h[1][:n], 1e-300)
        assert rel.max() <= 1e-10, (v.name, rel.max())


def test_l1_ops_unaffected(bandmats):
    P, A = PROBLEMS["randspd_3000"], bandmats["randspd_3000"]
    x = np.random.default_rng(1).uniform(-1, 1, A.n)
    assert same_bits(A.spmv(x), O.spmv(P.A, x))


def test_stencil_defaults_to_csr_engine():
    assert cgvk.DeviceMatrix.from_csr(PROBLEMS["poisson3d_12"].A).engine()[0] == "csr"
