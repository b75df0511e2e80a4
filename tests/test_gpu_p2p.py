"""Peer-memory exchange of a row-partitioned solve (CGVK_GROUP_P2P,
csrc/cgvk_p2p.cuh): the chained kernels push boundary rows into the
neighbours' receive buffers and rank totals into every rank's table as
stamped 8-byte words; a boundary row fetches its halo entries when their
stamp arrives, the successor's prologue folds the totals in rank order — no
exchange launch, no finalize launch, no fence. On one GPU the ranks run in
this process (their peers' memory is this device's); every wait is then
already satisfied in stream order, so the tests exercise the data path and
the stamp protocol, not the overlap. Every rank's state must be
bit-identical to the oracle restatement with partitioned dots
(ORC_DOT_PART), as the copy transport is."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1905_01549_b200 import cgvk, problems as pb
from paper_1905_01549_b200.cgvk import Precond, Variant, Vec

from helpers import ALL_VARIANTS
from test_gpu_group import compare

pytestmark = pytest.mark.gpu

PROBLEMS = {
    "poisson3d_12_slabs": (lambda: pb.poisson3d(12), 144),
    "poisson3d_16_slabs": (lambda: pb.poisson3d(16), 256),
}
_cache = {}


def problem(name):
    if name not in _cache:
        make, align = PROBLEMS[name]
        _cache[name] = (pb.make_problem(name, make()), align)
    return _cache[name]


def make_group(P, align, nranks, variant, precond, cfg_kwargs=None, p2p=True):
    A = P.A
    lo = cgvk.partition_rows(A.n, nranks, align)
    mats = [cgvk.RankMatrix(A.n, lo, r, *cgvk.local_rows(A, lo, r)) for r in range(nranks)]
    comm = cgvk.Comm(nranks)
    cfg = cgvk.VariantConfig.make(variant)
    for k, v in (cfg_kwargs or {}).items():
        setattr(cfg, k, v)
    g = cgvk.Group(comm, mats, cfg, precond, [P.b[lo[r]:lo[r + 1]] for r in range(nranks)],
                   [P.x0[lo[r]:lo[r + 1]] for r in range(nranks)], p2p=p2p)
    return g, lo, mats, comm, cfg


@pytest.mark.parametrize("nranks", [2, 3, 4])
@pytest.mark.parametrize("precond", [Precond.IDENTITY, Precond.JACOBI])
@pytest.mark.parametrize("variant", ALL_VARIANTS)
def test_p2p_bit_exact_vs_partitioned_oracle(variant, precond, nranks):
    P, align = problem("poisson3d_12_slabs")
    g, lo, mats, comm, cfg = make_group(P, align, nranks, variant, precond)
    assert g.transport == "p2p"
    block, gmax, order = mats[0].reduction_config()
    o = O.Restatement(P.A, int(variant), int(precond), P.b, P.x0, dot=("part", block, gmax, lo, order))
    tag = f"p2p/{variant.name}/{precond.name}/P{nranks}"
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


@pytest.mark.parametrize("variant", ALL_VARIANTS)
def test_p2p_eight_ranks_batched_graphs(variant):
    """8 ranks (one NVSwitch box), graph-replayed batches of 8 and 1
    iterations (the chained graphs with their tails): bit-equal to single
    steps of the copy transport and to the partitioned oracle."""
    P, align = problem("poisson3d_16_slabs")
    g, lo, mats, comm, cfg = make_group(P, align, 8, variant, Precond.JACOBI)
    h, *_ = make_group(P, align, 8, variant, Precond.JACOBI, p2p=False)
    block, gmax, order = mats[0].reduction_config()
    o = O.Restatement(P.A, int(variant), 1, P.b, P.x0, dot=("part", block, gmax, lo, order))
    done = 0
    for k in (8, 1, 8, 3, 8):
        g.step(k)
        h.step(k)
        g.sync()
        h.sync()
        for _ in range(k):
            if o.state()["state"] == 0:
                o.step()
        done += k
        compare(g, o, f"p2p8/{variant.name} after {done}")
    for w in (Vec.X, Vec.R):
        assert np.array_equal(g.vector(w).view(np.int64), h.vector(w).view(np.int64))
    np.testing.assert_array_equal(g.solvers[0].history(), h.solvers[0].history())
    g.close()
    h.close()


@pytest.mark.parametrize("kw", [{"recompute_w": False}, {"nu_expression": cgvk.NuExpression.EXPANDED},
                                {"unsimplified_mu": True}])
@pytest.mark.parametrize("variant", [Variant.PIPE_PR, Variant.GV])
def test_p2p_ablations(variant, kw):
    if variant == Variant.GV and "recompute_w" in kw:
        pytest.skip("recompute_w is a pipe-PR flag")
    P, align = problem("poisson3d_12_slabs")
    try:
        g, lo, mats, comm, cfg = make_group(P, align, 3, variant, Precond.JACOBI, kw)
    except cgvk.InvalidArgument:
        pytest.skip("configuration not valid for this variant")
    block, gmax, order = mats[0].reduction_config()
    o = O.Restatement(P.A, int(variant), 1, P.b, P.x0, dot=("part", block, gmax, lo, order),
                      nu_expr=int(cfg.nu_expression), recompute_w=cfg.recompute_w,
                      unsimplified_mu=cfg.unsimplified_mu)
    for _ in range(10):
        g.step(1)
        g.sync()
        o.step()
    compare(g, o, f"p2p ablation {variant.name} {kw}")
    g.close()


def test_p2p_true_residual_and_tolerance_stop():
    """A solve to ||r|| <= 1e-8 ||b|| through the peer-memory iteration: the
    stop and the true residual equal the copy transport's."""
    P, align = problem("poisson3d_16_slabs")
    out = []
    for p2p in (True, False):
        g, *_ = make_group(P, align, 4, Variant.PIPE_PR, Precond.JACOBI, p2p=p2p)
        for s in g.solvers:
            s.set_tolerance(1e-8)
        g.step(400)
        g.sync()
        st = g.solvers[0]._status()[0]
        out.append((st.k, st.state, g.true_residual(), g.vector(Vec.X)))
        g.close()
    assert out[0][:3] == out[1][:3]
    assert out[0][1] == 3  # converged
    assert np.array_equal(out[0][3], out[1][3])


def test_p2p_rejects_scattered_send_rows():
    """A random-band partition sends scattered rows (not a prefix / suffix):
    the peer-memory transport refuses it loudly instead of falling back."""
    R = pb.make_problem("rs", pb.random_spd(3000, 13, 300, 7))
    with pytest.raises(cgvk.InvalidArgument, match="prefix"):
        make_group(R, 1, 2, Variant.HS, Precond.JACOBI)


@pytest.mark.parametrize("variant", [Variant.HS, Variant.GV, Variant.PIPE_PR])
def test_p2p_nccl_single_rank(variant):
    """The multi-process set-up path (an NCCL communicator: the window is a
    plain cudaMalloc exported with cudaIpcGetMemHandle, the rank blobs are
    all-gathered through NCCL) on the one rank a single GPU admits."""
    P, align = problem("poisson3d_12_slabs")
    A = P.A
    lo = cgvk.partition_rows(A.n, 1, align)
    mats = [cgvk.RankMatrix(A.n, lo, 0, *cgvk.local_rows(A, lo, 0))]
    comm = cgvk.Comm(1, 0, 0, cgvk.nccl_unique_id())
    g = cgvk.Group(comm, mats, cgvk.VariantConfig.make(variant), Precond.JACOBI, [P.b], [P.x0], p2p=True)
    assert g.transport == "p2p"
    block, gmax, order = mats[0].reduction_config()
    o = O.Restatement(A, int(variant), 1, P.b, P.x0, dot=("part", block, gmax, lo, order))
    for k in (1, 8, 3):
        g.step(k)
        g.sync()
        for _ in range(k):
            if o.state()["state"] == 0:
                o.step()
        compare(g, o, f"p2p nccl1/{variant.name} k={o.state()['k']}")
    g.close()
    comm.close()


def test_p2p_wait_that_gives_up_is_reported(monkeypatch):
    """A rank whose wait gives up (here: an injected link latency longer than
    the 2 s bound) finishes its kernels and reports CGVK_ECUDA at the next
    sync instead of hanging the GPU."""
    monkeypatch.setenv("CGVK_P2P_DELAY_NS", str(int(2.1e9)))  # (an int: < 2^31 ns)
    P, align = problem("poisson3d_12_slabs")
    g, *_ = make_group(P, align, 1, Variant.HS, Precond.JACOBI)
    monkeypatch.delenv("CGVK_P2P_DELAY_NS")
    g.step(1)
    with pytest.raises(cgvk.CgvkError, match="gave up"):
        g.sync()
    g.close()


@pytest.mark.parametrize("kind", ["local", "nccl"])
def test_communicator_released_before_its_groups(kind):
    """The caller may release the communicator before the groups made over
    it (interpreter shutdown does, in any order): the groups keep it alive."""
    P, align = problem("poisson3d_12_slabs")
    A = P.A
    lo = cgvk.partition_rows(A.n, 1, align)
    mats = [cgvk.RankMatrix(A.n, lo, 0, *cgvk.local_rows(A, lo, 0))]
    comm = cgvk.Comm(1, 0, 0, cgvk.nccl_unique_id()) if kind == "nccl" else cgvk.Comm(1)
    g = cgvk.Group(comm, mats, cgvk.VariantConfig.make(Variant.PIPE_PR), Precond.JACOBI, [P.b], [P.x0],
                   p2p=True)
    comm.close()
    g.step(3)
    g.sync()
    assert g.solvers[0].k == 3
    g.close()


@pytest.mark.parametrize("cfg,nranks", [("p64", 8), ("p128", 2)])
@pytest.mark.parametrize("variant", [Variant.HS, Variant.PR, Variant.GV, Variant.PIPE_PR])
def test_p2p_baseline_shards_equal_copy_transport(cfg, nranks, variant):
    """BASELINE-size shards (P64 over 8 ranks: 16 boundary tiles per side of a
    128-tile rank; P128 over 2: 64 of 4096): 24 iterations through the peer
    transport give the copy transport's bits — histories and x."""
    P = pb.config_problem(cfg)
    plane = {"p64": 64 * 64, "p128": 128 * 128}[cfg]
    out = []
    for p2p in (True, False):
        g, *_ = make_group(P, plane, nranks, variant, Precond.JACOBI, p2p=p2p)
        assert g.transport == ("p2p" if p2p else "local")
        g.step(24)
        g.sync()
        out.append((g.solvers[0].history(), g.vector(Vec.X)))
        g.close()
    assert np.array_equal(out[0][0].view(np.int64), out[1][0].view(np.int64))
    assert np.array_equal(out[0][1].view(np.int64), out[1][1].view(np.int64))


@pytest.mark.parametrize("nranks", [2, 8])
@pytest.mark.parametrize("precond", [Precond.IDENTITY, Precond.JACOBI])
@pytest.mark.parametrize("variant", [Variant.M, Variant.PR])
def test_p2p_one_kernel_iteration(variant, precond, nranks, monkeypatch):
    """PR / M ranks that fit L2 run ONE kernel per rank and iteration (PrF,
    csrc/cgvk_variants.cuh: the previous iteration's r~, s, p pushed to the
    neighbours, p re-formed at the halo columns too): bit-equal to the
    two-kernel peer schedule (CGVK_FUSE_PEER=0) and the partitioned oracle,
    through odd and even graph batches."""
    P, align = problem("poisson3d_16_slabs")
    g, lo, mats, comm, cfg = make_group(P, align, nranks, variant, precond)
    monkeypatch.setenv("CGVK_FUSE_PEER", "0")
    h, *_ = make_group(P, align, nranks, variant, precond)
    monkeypatch.delenv("CGVK_FUSE_PEER")
    assert g.transport == "p2p" and h.transport == "p2p"
    assert g.solvers[0].launches_per_iter() == nranks and h.solvers[0].launches_per_iter() == 2 * nranks
    block, gmax, order = mats[0].reduction_config()
    o = O.Restatement(P.A, int(variant), int(precond), P.b, P.x0, dot=("part", block, gmax, lo, order))
    done = 0
    for k in (1, 1, 8, 3, 2, 9):
        g.step(k)
        h.step(k)
        g.sync()
        h.sync()
        for _ in range(k):
            if o.state()["state"] == 0:
                o.step()
        done += k
        compare(g, o, f"p2p-one-kernel/{variant.name}/{precond.name}/P{nranks} after {done}")
        for w in (Vec.X, Vec.R, Vec.P, Vec.S):
            assert np.array_equal(g.vector(w).view(np.int64), h.vector(w).view(np.int64)), (w, done)
    g.close()
    h.close()
