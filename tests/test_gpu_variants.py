"""The reference's own variant tests (proj/tests/test_variants.cpp,
test_sparse_matrix.cpp, test_preconditioner.cpp), restated against the GPU
path through the C-ABI, plus the edge cases the reference handles: exact
zero residuals, terminated solvers, dimension and Jacobi errors, n = 0."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1905_01549_b200 import cgvk, problems as pb
from paper_1905_01549_b200.cgvk import Precond, State, Variant, Vec

from helpers import lockstep, same_bits

pytestmark = pytest.mark.gpu

ALL = list(Variant)


def identity(n):
    return pb.CSR(n, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int64), np.ones(n))


def rvec(n, seed):
    return np.random.default_rng(seed).uniform(-1, 1, n)


def dense_csr(M):
    n = M.shape[0]
    rp, ci, va = [0], [], []
    for i in range(n):
        for j in range(n):
            if M[i, j] != 0.0:
                ci.append(j)
                va.append(M[i, j])
        rp.append(len(ci))
    return pb.CSR(n, np.array(rp, np.int64), np.array(ci, np.int64), np.array(va))


def random_spd_dense(n, kappa, seed):
    """SPD with a uniform spectrum in [1/kappa, 1] (oracles.cpp:19-37 recipe,
    numpy QR instead of Eigen), mirrored upper triangle for bit-symmetry."""
    rng = np.random.default_rng(seed)
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = np.linspace(1.0 / kappa, 1.0, n)
    M = (Q * lam) @ Q.T
    return np.triu(M) + np.triu(M, 1).T


@pytest.mark.parametrize("v", ALL)
def test_initialize_on_identity(v):
    """A=I, x0=0: p0 = b, s0 = b, alpha0 = 1 (test_variants.cpp:37-49)."""
    A = cgvk.DeviceMatrix.from_csr(identity(8))
    b = rvec(8, 1)
    s = cgvk.initialize(cgvk.VariantConfig.make(v), A, Precond.IDENTITY, b, np.zeros(8))
    assert s.status.running()
    assert same_bits(s.vector(Vec.P), b) and same_bits(s.vector(Vec.S), b)
    assert s.scalars()["alpha"] == 1.0


def test_exact_initial_guess_converges():
    """test_variants.cpp:51-60."""
    A = cgvk.DeviceMatrix.from_csr(identity(4))
    b = np.array([1.0, 2.0, 3.0, 4.0])
    s = cgvk.initialize(cgvk.VariantConfig.make(Variant.HS), A, Precond.IDENTITY, b, b.copy())
    st = s.status
    assert st.state == State.CONVERGED and st.criterion == cgvk.ConvergedBy.ZERO_RESIDUAL
    assert s.scalars()["nu"] == 0.0
    with pytest.raises(cgvk.LogicError):  # step() on a terminated solver
        s.step()


@pytest.mark.parametrize("v", ALL)
def test_one_step_on_identity_is_exact(v):
    """test_variants.cpp:74-89."""
    A = cgvk.DeviceMatrix.from_csr(identity(10))
    b = rvec(10, 2)
    s = cgvk.initialize(cgvk.VariantConfig.make(v), A, Precond.IDENTITY, b, np.zeros(10))
    cgvk.step(s)
    assert s.k == 1
    assert same_bits(s.x, b)
    assert np.linalg.norm(s.r) == 0.0
    assert s.status.state == State.CONVERGED


def test_pipelined_prediction_exact_zero():
    """test_variants.cpp:91-102: w'_1 = w0 - alpha0 u0 = 0 bit-exactly."""
    A = cgvk.DeviceMatrix.from_csr(identity(6))
    b = rvec(6, 9)
    s = cgvk.initialize(cgvk.VariantConfig.make(Variant.PIPE_PR), A, Precond.IDENTITY, b,
                        np.zeros(6))
    assert same_bits(s.vector(Vec.U), b)
    cgvk.step(s)
    assert np.all(s.vector(Vec.W) == 0.0)
    assert s.status.state == State.CONVERGED


def test_gv_initialization():
    """test_variants.cpp:104-111: u0 = A s~0 = b, w0 = b."""
    A = cgvk.DeviceMatrix.from_csr(identity(5))
    b = rvec(5, 4)
    s = cgvk.initialize(cgvk.VariantConfig.make(Variant.GV), A, Precond.IDENTITY, b, np.zeros(5))
    assert same_bits(s.vector(Vec.U), b) and same_bits(s.vector(Vec.W), b)


def test_cg_cg_first_step_bit_identical_to_hs():
    """test_variants.cpp:113-125."""
    A = cgvk.DeviceMatrix.from_csr(identity(12))
    b = rvec(12, 5)
    hs = cgvk.initialize(cgvk.VariantConfig.make(Variant.HS), A, Precond.IDENTITY, b, np.zeros(12))
    cg = cgvk.initialize(cgvk.VariantConfig.make(Variant.CG_CG), A, Precond.IDENTITY, b,
                         np.zeros(12))
    cgvk.step(hs)
    cgvk.step(cg)
    assert same_bits(hs.x, cg.x) and same_bits(hs.r, cg.r)
    assert hs.status.state == cg.status.state


def test_hs_tracks_extended_precision_cg():
    """test_variants.cpp:127-152 (512-bit MPFR oracle there; a float128-free
    restatement here: np.longdouble CG on the same shifted Hilbert matrix)."""
    M = np.array([[1.0 / (i + j + 1) + (0.1 if i == j else 0.0) for j in range(4)]
                  for i in range(4)])
    A = cgvk.DeviceMatrix.from_csr(dense_csr(M))
    b = np.array([1.0, -0.5, 0.25, 2.0])
    s = cgvk.initialize(cgvk.VariantConfig.make(Variant.HS), A, Precond.IDENTITY, b, np.zeros(4))
    Ml = M.astype(np.longdouble)
    x = np.zeros(4, np.longdouble)
    r = b.astype(np.longdouble)
    p = r.copy()
    for _ in range(4):
        Ap = Ml @ p
        a = (r @ r) / (p @ Ap)
        x = x + a * p
        rn = r - a * Ap
        p = rn + ((rn @ rn) / (r @ r)) * p
        r = rn
        cgvk.step(s)
        assert s.status.running()
        assert np.linalg.norm(s.x - x.astype(np.float64)) <= 1e-12 * np.linalg.norm(x.astype(np.float64))


def test_cg_cg_scalars_match_hs():
    """test_variants.cpp:154-169 (random SPD n=50, kappa=100)."""
    Ad = dense_csr(random_spd_dense(50, 100.0, 31))
    A = cgvk.DeviceMatrix.from_csr(Ad)
    b = rvec(50, 32)
    hs = cgvk.initialize(cgvk.VariantConfig.make(Variant.HS), A, Precond.IDENTITY, b, np.zeros(50))
    cg = cgvk.initialize(cgvk.VariantConfig.make(Variant.CG_CG), A, Precond.IDENTITY, b,
                         np.zeros(50))
    for _ in range(10):
        cgvk.step(hs)
        cgvk.step(cg)
        assert hs.status.running() and cg.status.running()
        a, c = hs.scalars(), cg.scalars()
        assert c["alpha"] == pytest.approx(a["alpha"], rel=1e-10)
        assert c["beta"] == pytest.approx(a["beta"], rel=1e-10)


def test_gv_error_tracks_hs():
    """test_variants.cpp:171-192."""
    Md = random_spd_dense(50, 100.0, 77)
    Ad = dense_csr(Md)
    A = cgvk.DeviceMatrix.from_csr(Ad)
    xs = np.full(50, 1.0 / np.sqrt(50.0))
    b = O.spmv(Ad, xs)
    hs = cgvk.initialize(cgvk.VariantConfig.make(Variant.HS), A, Precond.IDENTITY, b, np.zeros(50))
    gv = cgvk.initialize(cgvk.VariantConfig.make(Variant.GV), A, Precond.IDENTITY, b, np.zeros(50))
    for _ in range(10):
        cgvk.step(hs)
        cgvk.step(gv)
        eh, eg = xs - hs.x, xs - gv.x
        err_h, err_g = np.sqrt(eh @ (Md @ eh)), np.sqrt(eg @ (Md @ eg))
        assert abs(err_g - err_h) <= 1e-8 * err_h


@pytest.mark.parametrize("v,plain,prec", [(Variant.HS, 4, 5), (Variant.CG_CG, 5, 6),
                                          (Variant.M, 4, 6), (Variant.PR, 4, 6),
                                          (Variant.GV, 7, 10), (Variant.PIPE_PR_M, 6, 10),
                                          (Variant.PIPE_PR, 6, 10)])
def test_allocated_vectors_match_table1(v, plain, prec):
    """test_variants.cpp:194-217 (Table 1 'mem' column)."""
    Ad = dense_csr(random_spd_dense(20, 10.0, 8))
    A = cgvk.DeviceMatrix.from_csr(Ad)
    b = rvec(20, 6)
    s0 = cgvk.initialize(cgvk.VariantConfig.make(v), A, Precond.IDENTITY, b, np.zeros(20))
    s1 = cgvk.initialize(cgvk.VariantConfig.make(v), A, Precond.JACOBI, b, np.zeros(20))
    assert s0.allocated_vectors() == plain and s1.allocated_vectors() == prec
    assert sum(s1.has_vector(w) for w in Vec) == prec


@pytest.mark.parametrize("v", ALL)
def test_one_traversal_of_a_per_iteration(v):
    """test_variants.cpp:219-241 via SolverStats."""
    Ad = dense_csr(random_spd_dense(30, 1e3, 13))
    A = cgvk.DeviceMatrix.from_csr(Ad)
    b = rvec(30, 14)
    s = cgvk.initialize(cgvk.VariantConfig.make(v), A, Precond.IDENTITY, b, np.zeros(30))
    base = s.stats()
    for _ in range(5):
        cgvk.step(s)
    assert s.status.running()
    st = s.stats()
    dsp, dbl = st["spmv_calls"] - base["spmv_calls"], st["block_spmv_calls"] - base["block_spmv_calls"]
    if v in (Variant.PIPE_PR, Variant.PIPE_PR_M):
        assert dsp == 0 and dbl == 5
    else:
        assert dsp == 5 and dbl == 0


@pytest.mark.parametrize("v,scal", [(Variant.HS, 2), (Variant.CG_CG, 2), (Variant.M, 3),
                                    (Variant.PR, 4), (Variant.GV, 2), (Variant.PIPE_PR_M, 3),
                                    (Variant.PIPE_PR, 4)])
def test_reductions_per_iteration_match_table1(v, scal):
    """test_variants.cpp:243-263 (Table 1 'scal' column)."""
    Ad = dense_csr(random_spd_dense(30, 1e3, 17))
    A = cgvk.DeviceMatrix.from_csr(Ad)
    b = rvec(30, 18)
    s = cgvk.initialize(cgvk.VariantConfig.make(v), A, Precond.IDENTITY, b, np.zeros(30))
    base = s.stats()["reductions"]
    cgvk.step(s)
    assert s.status.running()
    assert s.stats()["reductions"] - base == scal


def test_recompute_w_off_carries_prediction():
    """test_variants.cpp:284-299."""
    Ad = dense_csr(random_spd_dense(16, 100.0, 2))
    A = cgvk.DeviceMatrix.from_csr(Ad)
    b = rvec(16, 5)
    cfg = cgvk.VariantConfig.make(Variant.PIPE_PR)
    cfg.recompute_w = False
    st = cgvk.initialize(cfg, A, Precond.IDENTITY, b, np.zeros(16))
    ref = cgvk.initialize(cgvk.VariantConfig.make(Variant.PIPE_PR), A, Precond.IDENTITY, b,
                          np.zeros(16))
    cgvk.step(st)
    cgvk.step(ref)
    ar = A.spmv(ref.r)
    assert same_bits(ref.vector(Vec.W), ar)
    assert not same_bits(st.vector(Vec.W), ar)


def test_meurant_from_pr_stepper_reproduces_m():
    """test_variants.cpp:319-335."""
    Ad = dense_csr(random_spd_dense(32, 100.0, 4))
    A = cgvk.DeviceMatrix.from_csr(Ad)
    b = rvec(32, 7)
    cfg = cgvk.VariantConfig.make(Variant.PR)
    cfg.nu_expression = cgvk.NuExpression.MEURANT
    a = cgvk.initialize(cfg, A, Precond.IDENTITY, b, np.zeros(32))
    m = cgvk.initialize(cgvk.VariantConfig.make(Variant.M), A, Precond.IDENTITY, b, np.zeros(32))
    for _ in range(20):
        cgvk.step(a)
        cgvk.step(m)
        assert a.status.running()
        assert same_bits(a.x, m.x)
        assert a.scalars()["nu_prime"] == m.scalars()["nu_prime"]


def test_expanded_equals_simplified_unpreconditioned():
    """test_variants.cpp:337-354."""
    Ad = dense_csr(random_spd_dense(24, 100.0, 6))
    A = cgvk.DeviceMatrix.from_csr(Ad)
    b = rvec(24, 8)
    cfg = cgvk.VariantConfig.make(Variant.PR)
    cfg.nu_expression = cgvk.NuExpression.EXPANDED
    a = cgvk.initialize(cfg, A, Precond.IDENTITY, b, np.zeros(24))
    c = cgvk.initialize(cgvk.VariantConfig.make(Variant.PR), A, Precond.IDENTITY, b, np.zeros(24))
    for _ in range(20):
        cgvk.step(a)
        cgvk.step(c)
        assert a.status.running()
        assert a.scalars()["nu_prime"] == c.scalars()["nu_prime"]
        assert same_bits(a.x, c.x)


ABLATIONS = [
    (Variant.PR, {"nu_expression": cgvk.NuExpression.EXPANDED}),
    (Variant.PR, {"recompute_nu": False}),
    (Variant.PIPE_PR, {"recompute_w": False}),
    (Variant.PIPE_PR, {"nu_expression": cgvk.NuExpression.EXPANDED}),
    (Variant.PIPE_PR, {"recompute_nu": False}),
    (Variant.M, {"track_delta": True}),
    (Variant.PIPE_PR_M, {"track_delta": True}),
    (Variant.CG_CG, {"unsimplified_mu": True}),
    (Variant.GV, {"unsimplified_mu": True}),
]


@pytest.mark.parametrize("precond", [Precond.IDENTITY, Precond.JACOBI])
@pytest.mark.parametrize("v,kw", ABLATIONS, ids=lambda x: str(x))
def test_ablation_flags_bit_exact(v, kw, precond):
    """every ablation flag on the device, bit-exact vs the
    GPU-order oracle."""
    P = pb.make_problem("vc", pb.varcoef3d(10))
    A = cgvk.DeviceMatrix.from_csr(P.A)
    lockstep(P.A, A, v, precond, P.b, P.x0, steps=20, cfg_kwargs=kw, check_vectors_every=4)


def test_predictor_scalars_positive_while_running():
    """test_variants.cpp:265-282 (model problem -> var-coef stand-in)."""
    P = pb.make_problem("vc", pb.varcoef3d(8, seed=3, sigma=1.0))
    A = cgvk.DeviceMatrix.from_csr(P.A)
    for v in (Variant.M, Variant.PR, Variant.PIPE_PR_M, Variant.PIPE_PR):
        s = cgvk.initialize(cgvk.VariantConfig.make(v), A, Precond.IDENTITY, P.b, P.x0)
        for _ in range(300):
            if not s.status.running():
                break
            cgvk.step(s)
            if s.status.running():
                sc = s.scalars()
                assert sc["nu_prime"] > 0.0 and sc["mu"] > 0.0


# ----------------------------------------------------------- L1 / errors

def test_spmv_identity_and_diagonal():
    """test_sparse_matrix.cpp:30-45."""
    A = cgvk.DeviceMatrix.from_csr(identity(17))
    x = rvec(17, 1)
    assert same_bits(A.spmv(x), x)
    d = np.array([2.0, -3.5, 0.25, 7.0])
    D = cgvk.DeviceMatrix(4, np.arange(5), np.arange(4), d)
    assert same_bits(D.spmv(np.array([1.0, 2.0, 4.0, -1.0])), d * np.array([1.0, 2.0, 4.0, -1.0]))


def test_spmv_dense_row_and_ragged():
    """A dense matrix (rows longer than a pipeline chunk) and empty rows."""
    rng = np.random.default_rng(4)
    M = rng.uniform(-1, 1, (300, 300))
    M[5, :] = 0.0
    Ad = dense_csr(M)
    A = cgvk.DeviceMatrix.from_csr(Ad)
    x = rng.uniform(-1, 1, 300)
    assert same_bits(A.spmv(x), O.spmv(Ad, x))
    y1, y2 = A.block_spmv(x, 2 * x)
    assert same_bits(y1, O.spmv(Ad, x)) and same_bits(y2, O.spmv(Ad, 2 * x))


def test_dimension_and_csr_errors():
    A = cgvk.DeviceMatrix.from_csr(identity(4))
    with pytest.raises(cgvk.InvalidArgument):
        A.spmv(np.ones(3))
    with pytest.raises(cgvk.InvalidArgument):  # columns not increasing
        cgvk.DeviceMatrix(2, np.array([0, 2, 3]), np.array([1, 0, 1]), np.ones(3))
    with pytest.raises(cgvk.InvalidArgument):  # column out of range
        cgvk.DeviceMatrix(2, np.array([0, 1, 2]), np.array([0, 2]), np.ones(2))
    with pytest.raises(cgvk.InvalidArgument):  # row_ptr not monotone
        cgvk.DeviceMatrix(2, np.array([0, 2, 1]), np.array([0, 1]), np.ones(2))
    with pytest.raises(cgvk.InvalidArgument):  # not bit-symmetric
        cgvk.DeviceMatrix(2, np.array([0, 2, 4]), np.array([0, 1, 0, 1]),
                          np.array([2.0, 1.0, 0.5, 2.0]), check_symmetric=True)
    with pytest.raises(cgvk.InvalidArgument):
        cgvk.initialize(cgvk.VariantConfig.make(Variant.HS), A, Precond.IDENTITY, np.ones(3),
                        np.zeros(4))


def test_jacobi_rejects_missing_or_nonpositive_diagonal():
    """test_preconditioner.cpp:31-42 (+ 20-29 values)."""
    A = cgvk.DeviceMatrix(2, np.array([0, 2, 4]), np.array([0, 1, 0, 1]),
                          np.array([2.0, 1.0, 1.0, 4.0]))
    assert list(A.jacobi()) == [0.5, 0.25]
    assert list(A.precond_apply(Precond.JACOBI, np.array([3.0, 8.0]))) == [1.5, 2.0]
    missing = cgvk.DeviceMatrix(2, np.array([0, 1, 2]), np.array([1, 0]), np.ones(2))
    with pytest.raises(cgvk.InvalidArgument):
        missing.jacobi()
    neg = cgvk.DeviceMatrix(2, np.array([0, 1, 2]), np.array([0, 1]), np.array([-1.0, 1.0]))
    with pytest.raises(cgvk.InvalidArgument):
        cgvk.initialize(cgvk.VariantConfig.make(Variant.HS), neg, Precond.JACOBI, np.ones(2),
                        np.zeros(2))


def test_empty_system():
    A = cgvk.DeviceMatrix(0, np.zeros(1, np.int64), np.zeros(0, np.int64), np.zeros(0))
    s = cgvk.initialize(cgvk.VariantConfig.make(Variant.PR), A, Precond.IDENTITY, np.zeros(0),
                        np.zeros(0))
    assert s.status.state == State.CONVERGED
    with pytest.raises(cgvk.LogicError):
        s.step()


@pytest.mark.parametrize("v", ALL)
def test_breakdown_reported_not_thrown(v):
    """An indefinite matrix drives nu/mu/nu' non-positive: the status says
    Breakdown with the reference's reason, bit-exact vs the oracle."""
    M = np.diag([1.0, 2.0, -3.0, 4.0, -0.5, 1.5])
    Ad = dense_csr(M)
    A = cgvk.DeviceMatrix.from_csr(Ad)
    b = np.array([1.0, 1.0, 1.0, 1.0, 1.0, 1.0])
    lockstep(Ad, A, v, Precond.IDENTITY, b, np.zeros(6), steps=10)


@pytest.mark.parametrize("v", ALL)
def test_tolerance_stop(v):
    P = pb.make_problem("p2", pb.poisson2d(40))
    A = cgvk.DeviceMatrix.from_csr(P.A)
    s = cgvk.initialize(cgvk.VariantConfig.make(v), A, Precond.JACOBI, P.b, P.x0)
    s.set_tolerance(1e-8)
    s.step(5000)
    s.sync()
    st = s.status
    assert st.state == State.CONVERGED and st.criterion == cgvk.ConvergedBy.TOLERANCE
    o = O.Restatement(P.A, int(v), 1, P.b, P.x0, dot=("tree",) + A.reduction_config())
    taken, upd, _ = o.solve(P.b, 5000, 1e-8)
    assert s.k == taken
    assert same_bits(s.x, o.vector(0))
    x, status, k = cgvk.solve(A, cgvk.VariantConfig.make(v), Precond.JACOBI, P.b, P.x0, 5000, 1e-8)
    assert k == taken and same_bits(x, o.vector(0))
    x, status, k = cgvk.solve(A, cgvk.VariantConfig.make(v), Precond.JACOBI, P.b, P.x0, 7)
    assert k == 7 and status.state == State.MAX_ITERATIONS


@pytest.mark.parametrize("v", ALL)
@pytest.mark.parametrize("case", ["mu0", "nonfinite_nu0"])
def test_initialize_settles_status(v, case):
    """initialize()'s own checks (src/variants.cpp:383, 389): mu0 <= 0 on an
    indefinite matrix, a non-finite nu0 from a NaN in b. Creation is
    stream-ordered — every kernel is enqueued and the device restores what
    the reference never computed — so status, scalars, counters and every
    vector must be exactly the reference's."""
    M = np.diag([1.0, -3.0, 0.5, 1.0])
    Ad = dense_csr(M)
    A = cgvk.DeviceMatrix.from_csr(Ad)
    b = np.ones(4)
    if case == "nonfinite_nu0":
        b[2] = np.nan
    s, o = lockstep(Ad, A, v, Precond.IDENTITY, b, np.zeros(4), steps=0)
    st = s.status
    assert st.state == State.BREAKDOWN
    assert st.breakdown == (cgvk.Breakdown.MU_NONPOSITIVE if case == "mu0" else cgvk.Breakdown.NON_FINITE)
    with pytest.raises(cgvk.LogicError):
        cgvk.step(s)


@pytest.mark.parametrize("v", ALL)
@pytest.mark.parametrize("precond", [Precond.IDENTITY, Precond.JACOBI])
def test_async_path_matches_synchronous(v, precond):
    """cgvk_solver_create (stream-ordered), step(n) and the asynchronous x
    download with one sync at the end give the same bits as step-by-step
    synchronous use; solvers created back to back share nothing."""
    P = pb.make_problem("p2", pb.poisson2d(30))
    A = cgvk.DeviceMatrix.from_csr(P.A)
    cfg = cgvk.VariantConfig.make(v)
    outs = [np.empty(A.n) for _ in range(3)]
    for o in outs:
        cgvk.host_register(o)
    try:
        ss = [cgvk.initialize(cfg, A, precond, P.b, P.x0) for _ in range(3)]
        for i, s in enumerate(ss):
            s.step(11 + i)
            s.x_async(outs[i])
        for s in ss:
            s.sync()
        for i, s in enumerate(ss):
            ref = cgvk.initialize(cfg, A, precond, P.b, P.x0)
            for _ in range(11 + i):
                cgvk.step(ref)
            assert same_bits(outs[i], ref.x) and s.k == ref.k == 11 + i
            assert gpu_state_equal(s, ref)
    finally:
        for o in outs:
            cgvk.host_unregister(o)


def gpu_state_equal(a, b):
    from helpers import gpu_state
    return gpu_state(a) == gpu_state(b)


def test_solver_after_orders_solves_without_changing_them():
    """cgvk_solver_after: a chain of solves ordered one after another (the
    bench's e2e order: each solve's steps after the previous one's, the
    previous download enqueued after the order point) gives the bits of the
    same solves run alone; ordering a solver after itself is a no-op."""
    P = pb.make_problem("p2", pb.poisson2d(30))
    A = cgvk.DeviceMatrix.from_csr(P.A)
    vs = [Variant.HS, Variant.GV, Variant.PIPE_PR, Variant.PR]
    outs = [np.empty(A.n) for _ in vs]
    for o in outs:
        cgvk.host_register(o)
    try:
        ss = []
        for i, v in enumerate(vs):
            s = cgvk.initialize(cgvk.VariantConfig.make(v), A, Precond.JACOBI, P.b, P.x0)
            if ss:
                s.after(ss[-1])
                ss[-1].x_async(outs[i - 1])
            s.after(s)
            s.step(17)
            ss.append(s)
        ss[-1].x_async(outs[-1])
        for s in ss:
            s.sync()
        for i, v in enumerate(vs):
            ref = cgvk.initialize(cgvk.VariantConfig.make(v), A, Precond.JACOBI, P.b, P.x0)
            ref.step(17)
            ref.sync()
            assert same_bits(outs[i], ref.x), v.name
            assert gpu_state_equal(ss[i], ref), v.name
    finally:
        for o in outs:
            cgvk.host_unregister(o)
