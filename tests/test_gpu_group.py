"""Row-partitioned solves on one GPU (the in-process 'local' transport runs
the data path of a P-GPU run: rank-local matrices in [own | halo] numbering,
halo exchanges, rank-ordered reductions). Every rank's state must be
bit-identical to the oracle restatement with partitioned dots
(ORC_DOT_PART: rank-local canonical trees summed in rank order) — all seven
variants x {none, Jacobi}, P = 2, 3, 4 — and its residual history must match
the single-GPU solve within the north-star tolerance."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1905_01549_b200 import cgvk, problems as pb
from paper_1905_01549_b200.cgvk import Precond, Variant, Vec

from helpers import ALL_VARIANTS, same_bits

pytestmark = pytest.mark.gpu

PROBLEMS = {
    "poisson3d_12_slabs": (lambda: pb.poisson3d(12), 144),
    "randspd_3000": (lambda: pb.random_spd(3000, 13, 300, 7), 1),
}
_cache = {}


def problem(name):
    if name not in _cache:
        make, align = PROBLEMS[name]
        _cache[name] = (pb.make_problem(name, make()), align)
    return _cache[name]


def make_group(P, align, nranks, variant, precond, cfg_kwargs=None):
    A = P.A
    lo = cgvk.partition_rows(A.n, nranks, align)
    mats = [cgvk.RankMatrix(A.n, lo, r, *cgvk.local_rows(A, lo, r)) for r in range(nranks)]
    comm = cgvk.Comm(nranks)
    cfg = cgvk.VariantConfig.make(variant)
    for k, v in (cfg_kwargs or {}).items():
        setattr(cfg, k, v)
    bs = [P.b[lo[r]:lo[r + 1]] for r in range(nranks)]
    xs = [P.x0[lo[r]:lo[r + 1]] for r in range(nranks)]
    g = cgvk.Group(comm, mats, cfg, precond, bs, xs)
    return g, lo, mats, comm, cfg


def compare(g, o, where):
    ost = o.state()
    for s in g.solvers:
        st, sc, stats = s._status()
        assert st.k == ost["k"] and st.state == ost["state"], where
        assert st.breakdown == ost["breakdown"] and st.criterion == ost["criterion"], where
        assert {k: getattr(stats, k) for k in ost["stats"]} == ost["stats"], where
        for name, ov in ost["scalars"].items():
            gv = getattr(sc, name)
            assert same_bits(np.float64(gv), np.float64(ov)) or (np.isnan(gv) and np.isnan(ov)), \
                f"{where} {name}"
    for w in Vec:
        ov = o.vector(int(w))
        try:
            gv = g.vector(w)
        except cgvk.InvalidArgument:
            gv = None
        assert same_bits(gv, ov), f"{where} vector {w.name}"


@pytest.mark.parametrize("nranks", [2, 3, 4])
@pytest.mark.parametrize("precond", [Precond.IDENTITY, Precond.JACOBI])
@pytest.mark.parametrize("variant", ALL_VARIANTS)
@pytest.mark.parametrize("name", list(PROBLEMS))
def test_group_bit_exact_vs_partitioned_oracle(name, variant, precond, nranks):
    P, align = problem(name)
    g, lo, mats, comm, cfg = make_group(P, align, nranks, variant, precond)
    block, gmax, order = mats[0].reduction_config()
    o = O.Restatement(P.A, int(variant), int(precond), P.b, P.x0, dot=("part", block, gmax, lo, order))
    tag = f"{name}/{variant.name}/{precond.name}/P{nranks}"
    compare(g, o, tag + " init")
    for k in range(1, 16):
        if o.state()["state"] != 0:
            break
        g.step(1)
        g.sync()
        o.step()
        if k % 5 == 0 or o.state()["state"] != 0:
            compare(g, o, f"{tag} k={k}")
    g.close()


@pytest.mark.parametrize("variant", [Variant.HS, Variant.PR, Variant.GV, Variant.PIPE_PR])
def test_group_batched_graph_and_true_residual(variant):
    """Graph-replayed batches (8- and 1-iteration graphs with exchanges) land
    on the same bits as single steps; the group true residual equals the
    oracle's; histories agree with the single-GPU solve within 1e-10."""
    P, align = problem("poisson3d_12_slabs")
    g, lo, mats, comm, cfg = make_group(P, align, 3, variant, Precond.JACOBI)
    h, _, _, _, _ = make_group(P, align, 3, variant, Precond.JACOBI)
    g.step(19)
    g.sync()
    for _ in range(19):
        h.step(1)
        h.sync()
    assert same_bits(g.vector(Vec.X), h.vector(Vec.X))
    block, gmax, order = mats[0].reduction_config()
    o = O.Restatement(P.A, int(variant), 1, P.b, P.x0, dot=("part", block, gmax, lo, order))
    for _ in range(19):
        o.step()
    tmp = P.b - O.spmv(P.A, o.vector(0))
    want = np.sqrt(O.dot(tmp, tmp, ("part", block, gmax, lo, order)))
    assert g.true_residual() == want
    A1 = cgvk.DeviceMatrix.from_csr(P.A)
    s1 = cgvk.initialize(cfg, A1, Precond.JACOBI, P.b, P.x0)
    s1.step(19)
    s1.sync()
    np.testing.assert_allclose(g.solvers[0].history(), s1.history(), rtol=1e-10 if variant != Variant.GV else 1e-9)
    g.close()
    h.close()


@pytest.mark.parametrize("kw", [{"recompute_w": False}, {"nu_expression": cgvk.NuExpression.EXPANDED}])
def test_group_ablations(kw):
    P, align = problem("randspd_3000")
    g, lo, mats, comm, cfg = make_group(P, align, 2, Variant.PIPE_PR, Precond.JACOBI, kw)
    block, gmax, order = mats[0].reduction_config()
    o = O.Restatement(P.A, int(Variant.PIPE_PR), 1, P.b, P.x0, dot=("part", block, gmax, lo, order),
                      nu_expr=int(cfg.nu_expression), recompute_w=cfg.recompute_w)
    for _ in range(10):
        g.step(1)
        g.sync()
        o.step()
    compare(g, o, f"ablation {kw}")
    g.close()


@pytest.mark.parametrize("variant", [Variant.HS, Variant.CG_CG, Variant.PR, Variant.GV, Variant.PIPE_PR])
def test_nccl_transport_single_rank(variant):
    """The NCCL transport (dlopen'ed libnccl, ncclCommInitRank, the captured
    AllGather of the rank totals and the grouped halo Send/Recv) on a
    one-rank communicator — the only NCCL size one GPU admits — bit-exact vs
    the partitioned oracle, through several graph-replayed batches."""
    P, align = problem("poisson3d_12_slabs")
    A = P.A
    lo = cgvk.partition_rows(A.n, 1, align)
    mats = [cgvk.RankMatrix(A.n, lo, 0, *cgvk.local_rows(A, lo, 0))]
    comm = cgvk.Comm(1, 0, 0, cgvk.nccl_unique_id())
    assert comm.kind == "nccl"
    g = cgvk.Group(comm, mats, cgvk.VariantConfig.make(variant), Precond.JACOBI, [P.b], [P.x0])
    block, gmax, order = mats[0].reduction_config()
    o = O.Restatement(A, int(variant), 1, P.b, P.x0, dot=("part", block, gmax, lo, order))
    compare(g, o, f"nccl1/{variant.name} init")
    for k in (1, 8, 3):
        g.step(k)
        g.sync()
        for _ in range(k):
            if o.state()["state"] == 0:
                o.step()
        compare(g, o, f"nccl1/{variant.name} k={o.state()['k']}")
    g.close()
    comm.close()
