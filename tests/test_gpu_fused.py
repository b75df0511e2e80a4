"""PR / M, CG-CG, GV and pipe-PR (-M) as one kernel per iteration (PrF / CgF /
GvF / PprF, csrc/cgvk_variants.cuh) — the
schedule libcgvk picks for problems whose working set fits L2 — against the
two-kernel schedule (CGVK_FUSE=0) and the tree-order oracle: the same bits
in every state vector and scalar, whatever the step batching (1-iteration
and 8-iteration graphs alternate the buffer sets and control-block copies),
through breakdown, the tolerance stop and the ablation flags; for CG-CG / GV also
the deferred beta-recurrences (a vector read between steps materialises them
with a form-only launch, the next launch is step-only). The steps are
src/variants.cpp:207-234, :237-265, :267-298 and :303-350 in both schedules."""
import os

import numpy as np
import pytest

from paper_1905_01549_b200 import cgvk, problems as pb
from paper_1905_01549_b200.cgvk import Precond, State, Variant, Vec

from helpers import gpu_state, gpu_vectors, lockstep, same_bits

pytestmark = pytest.mark.gpu

PR_LIKE = [Variant.M, Variant.PR, Variant.CG_CG, Variant.GV, Variant.PIPE_PR, Variant.PIPE_PR_M]
PRECS = [Precond.IDENTITY, Precond.JACOBI]


class two_kernel:
    """Solvers created inside use the two-kernel schedule."""

    def __enter__(self):
        self.old = os.environ.get("CGVK_FUSE")
        os.environ["CGVK_FUSE"] = "0"

    def __exit__(self, *a):
        if self.old is None:
            del os.environ["CGVK_FUSE"]
        else:
            os.environ["CGVK_FUSE"] = self.old


def small_problem():
    """3-D Poisson, 15^3 = 3375 rows: several tiles, a partial last tile."""
    P = pb.make_problem("p15", pb.poisson3d(15), seed=3)
    return P.A, P.b, P.x0


def states_equal(a: cgvk.Solver, b: cgvk.Solver, where: str) -> None:
    ga, gb = gpu_state(a), gpu_state(b)
    assert ga["k"] == gb["k"] and ga["state"] == gb["state"] and ga["breakdown"] == gb["breakdown"], where
    assert ga["stats"] == gb["stats"], where
    for name, va in ga["scalars"].items():
        vb = gb["scalars"][name]
        assert same_bits(np.float64(va), np.float64(vb)) or (np.isnan(va) and np.isnan(vb)), f"{where}: {name}"
    va, vb = gpu_vectors(a), gpu_vectors(b)
    for w in va:
        assert same_bits(va[w], vb[w]), f"{where}: vector {w}"
    assert same_bits(a.history(), b.history()), f"{where}: residual history"


@pytest.mark.parametrize("v", PR_LIKE)
@pytest.mark.parametrize("precond", PRECS)
def test_schedule_is_one_launch_and_matches_two_kernel(v, precond):
    A, b, x0 = small_problem()
    Ad = cgvk.DeviceMatrix.from_csr(A)
    cfg = cgvk.VariantConfig.make(v)
    f = cgvk.initialize(cfg, Ad, precond, b, x0)
    with two_kernel():
        t = cgvk.initialize(cfg, Ad, precond, b, x0)
    assert f.launches_per_iter() == 1 and t.launches_per_iter() == 2
    states_equal(f, t, "init")
    # odd and even batches: 1-iteration graphs, the 8-iteration graph, mixes
    for n in (1, 1, 2, 3, 8, 9, 16, 5):
        f.step(n)
        t.step(n)
        states_equal(f, t, f"after +{n}")
    f.close()
    t.close()


@pytest.mark.parametrize("v", PR_LIKE)
@pytest.mark.parametrize("precond", PRECS)
def test_lockstep_with_oracle(v, precond):
    """Bit-identical to the tree-order restatement after every single step
    (every vector read back each step: exercises both buffer sets)."""
    A, b, x0 = small_problem()
    Ad = cgvk.DeviceMatrix.from_csr(A)
    s, _ = lockstep(A, Ad, v, precond, b, x0, 12)
    assert s.launches_per_iter() == 1
    s.close()


@pytest.mark.parametrize("v", PR_LIKE)
def test_two_kernel_schedule_still_bit_exact(v):
    """The schedule large problems run (P128, V256, R4M) on a small one."""
    A, b, x0 = small_problem()
    Ad = cgvk.DeviceMatrix.from_csr(A)
    with two_kernel():
        s, _ = lockstep(A, Ad, v, Precond.JACOBI, b, x0, 10, check_vectors_every=3)
        assert s.launches_per_iter() == 2
    s.close()


@pytest.mark.parametrize("v,kw", [(Variant.PR, {"recompute_nu": False}), (Variant.PR, {"track_delta": True}),
                                  (Variant.PR, {"nu_expression": 0}), (Variant.PR, {"nu_expression": 2}),
                                  (Variant.CG_CG, {"unsimplified_mu": True}),
                                  (Variant.GV, {"unsimplified_mu": True}),
                                  (Variant.PIPE_PR, {"recompute_nu": False}), (Variant.PIPE_PR, {"track_delta": True}),
                                  (Variant.PIPE_PR, {"nu_expression": 0})])
def test_ablation_flags(v, kw):
    A, b, x0 = small_problem()
    Ad = cgvk.DeviceMatrix.from_csr(A)
    cfg = cgvk.VariantConfig.make(v)
    for k_, v_ in kw.items():
        setattr(cfg, k_, v_)
    try:
        cfg.validate()
    except cgvk.InvalidArgument:
        pytest.skip("flag combination rejected by VariantConfig::validate")
    f = cgvk.initialize(cfg, Ad, Precond.JACOBI, b, x0)
    with two_kernel():
        t = cgvk.initialize(cfg, Ad, Precond.JACOBI, b, x0)
    assert f.launches_per_iter() == 1
    for n in (1, 4, 7):
        f.step(n)
        t.step(n)
        states_equal(f, t, f"{kw} after +{n}")
    s_, _ = lockstep(A, Ad, v, Precond.JACOBI, b, x0, 6, cfg_kwargs=kw)
    s_.close()
    f.close()
    t.close()


@pytest.mark.parametrize("v", PR_LIKE)
def test_solve_to_tolerance_and_beyond(v):
    """The tolerance stop lands on the same iteration with the same x; steps
    enqueued after it are device-side no-ops in both schedules."""
    A, b, x0 = small_problem()
    Ad = cgvk.DeviceMatrix.from_csr(A)
    cfg = cgvk.VariantConfig.make(v)
    f = cgvk.initialize(cfg, Ad, Precond.JACOBI, b, x0)
    with two_kernel():
        t = cgvk.initialize(cfg, Ad, Precond.JACOBI, b, x0)
    for s in (f, t):
        s.set_tolerance(1e-9)
        s.step(400)
    states_equal(f, t, "tolerance stop")
    assert f.status.state == State.CONVERGED and 0 < f.k < 400
    f.close()
    t.close()


def test_breakdown_on_indefinite_matrix():
    """An indefinite matrix breaks the recurrences down; both schedules report
    the same breakdown at the same step with the same vectors."""
    n = 700
    rng = np.random.default_rng(11)
    d = rng.uniform(0.5, 2.0, n) * np.where(np.arange(n) % 3 == 0, -1.0, 1.0)
    A = pb.CSR(n, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int64), d)
    b = rng.uniform(-1, 1, n)
    Ad = cgvk.DeviceMatrix.from_csr(A)
    for v in PR_LIKE:
        cfg = cgvk.VariantConfig.make(v)
        f = cgvk.initialize(cfg, Ad, Precond.IDENTITY, b, np.zeros(n))
        with two_kernel():
            t = cgvk.initialize(cfg, Ad, Precond.IDENTITY, b, np.zeros(n))
        for _ in range(30):
            if not f.status.running():
                break
            f.step(1)
            t.step(1)
            states_equal(f, t, f"{v.name} indefinite k={f.k}")
        assert f.status.state == t.status.state
        f.close()
        t.close()


def test_pipe_pr_without_recompute_w_keeps_two_kernels():
    """PprF is the paper's pipe-PR (recompute_w on); the stored-recurrence
    ablation runs the two-kernel schedule."""
    A, b, x0 = small_problem()
    Ad = cgvk.DeviceMatrix.from_csr(A)
    cfg = cgvk.VariantConfig.make(Variant.PIPE_PR)
    cfg.recompute_w = False
    s = cgvk.initialize(cfg, Ad, Precond.JACOBI, b, x0)
    assert s.launches_per_iter() == 2
    s.close()
