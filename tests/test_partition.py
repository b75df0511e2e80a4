"""Row partition and halo maps: the library's host logic
(cgvk_partition_rows / cgvk_halo_plan, no GPU needed) must equal the
independent CPU restatement in oracle/partition.py bit-for-bit; and a
2-process gloo run of the distributed data path (local numbering, halo
exchange, rank-ordered dots) reproduces the global SpMV and the partitioned
dot order exactly."""
import os
import socket

import numpy as np
import pytest

from oracle import oracle as O
from oracle import partition as OP
from paper_1905_01549_b200 import cgvk, problems as pb


CASES = [
    ("p3_16_slab", lambda: pb.poisson3d(16), 16 * 16),
    ("p2_40", lambda: pb.poisson2d(40), 40),
    ("vc_12_slab", lambda: pb.varcoef3d(12), 144),
    ("rspd_6000", lambda: pb.random_spd(6000, 13, 300, 7), 1),
]


@pytest.mark.parametrize("nparts", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("name,make,align", CASES, ids=[c[0] for c in CASES])
def test_partition_and_halo_maps_bit_exact(name, make, align, nparts):
    A = make()
    lo = cgvk.partition_rows(A.n, nparts, align)
    assert np.array_equal(lo, OP.partition_rows(A.n, nparts, align))
    assert lo[0] == 0 and lo[-1] == A.n and np.all(np.diff(lo) >= 0)
    for r in range(nparts):
        rp, ci, va = cgvk.local_rows(A, lo, r)
        got = cgvk.halo_plan(A.n, lo, r, rp, ci)
        want = OP.halo_maps(A, lo, r)
        for k in ("lower", "upper", "send_lo", "send_hi"):
            assert np.array_equal(got[k], want[k]), (r, k)
        # the neighbours agree on what crosses each boundary
        if r > 0:
            prev = OP.halo_maps(A, lo, r - 1)
            assert np.array_equal(got["lower"], prev["send_hi"] + lo[r - 1])
        if r + 1 < nparts:
            nxt = OP.halo_maps(A, lo, r + 1)
            assert np.array_equal(got["upper"], nxt["send_lo"] + lo[r + 1])


def test_z_slabs_of_the_baseline_grid():
    # P64 over 8 ranks: 8 planes each, one plane of halo per side
    n, plane = 64**3, 64 * 64
    lo = cgvk.partition_rows(n, 8, plane)
    assert np.array_equal(np.diff(lo), np.full(8, 8 * plane))


def test_halo_wider_than_a_neighbour_is_rejected():
    A = pb.poisson3d(8)  # +-64 coupling; 8-row blocks are thinner than that
    lo = cgvk.partition_rows(A.n, 64, 4)
    rp, ci, va = cgvk.local_rows(A, lo, 30)
    with pytest.raises(cgvk.InvalidArgument):
        cgvk.halo_plan(A.n, lo, 30, rp, ci)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        P = pb.make_problem("p3", pb.poisson3d(10))
        A = P.A
        lo = OP.partition_rows(A.n, world, 100)
        rp, ci, va, h = OP.local_matrix(A, lo, rank)
        m = int(lo[rank + 1] - lo[rank])
        x = P.x_star[lo[rank]:lo[rank + 1]]
        # halo exchange of x with the neighbours (the device protocol: pack the
        # rows the neighbour reads, receive into [own | lower | upper])
        xloc = np.zeros(m + len(h["lower"]) + len(h["upper"]))
        xloc[:m] = x
        reqs = []
        if rank > 0:
            reqs.append(dist.isend(torch.from_numpy(x[h["send_lo"]].copy()), rank - 1))
            buf_lo = torch.zeros(len(h["lower"]), dtype=torch.float64)
            reqs.append(dist.irecv(buf_lo, rank - 1))
        if rank + 1 < world:
            reqs.append(dist.isend(torch.from_numpy(x[h["send_hi"]].copy()), rank + 1))
            buf_hi = torch.zeros(len(h["upper"]), dtype=torch.float64)
            reqs.append(dist.irecv(buf_hi, rank + 1))
        for rq in reqs:
            rq.wait()
        if rank > 0:
            xloc[m:m + len(h["lower"])] = buf_lo.numpy()
        if rank + 1 < world:
            xloc[m + len(h["lower"]):] = buf_hi.numpy()
        y = OP.local_spmv(rp, ci, va, xloc)
        # rank-local canonical tree, gathered, summed in rank order
        part = O.dot(y, y, ("tree", 256, 1776, 0))
        parts = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, torch.tensor([part], dtype=torch.float64))
        tot = 0.0
        for t in parts:
            tot = tot + float(t.item())
        ys = [torch.zeros(int(lo[r + 1] - lo[r]), dtype=torch.float64) for r in range(world)]
        dist.all_gather(ys, torch.from_numpy(y))
        q.put((rank, np.concatenate([t.numpy() for t in ys]), tot))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_distributed_spmv_and_dot(world):
    """world_size-2 gloo: halo exchange + local SpMV == the global reference
    spmv bit-for-bit; rank-ordered dot == ORC_DOT_PART."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    P = pb.make_problem("p3", pb.poisson3d(10))
    y_ref = O.spmv(P.A, P.x_star)
    lo = OP.partition_rows(P.A.n, world, 100)
    want = O.dot(y_ref, y_ref, ("part", 256, 1776, lo, 0))
    for rank, y, tot in res:
        assert np.array_equal(y.view(np.int64), y_ref.view(np.int64))
        assert tot == want


def _worker_lib(rank, world, port, q):
    """The product's host logic on each process (libcgvk, no GPU): partition,
    halo plan and the device's local numbering (cgvk_rank_local_columns,
    exactly what cgvk_matrix_create_rank uploads); the halo moves as the
    peer-memory transport moves it (a rank's send rows are a prefix / suffix
    of its rows, landing at the neighbour's hbase + offset)."""
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        P = pb.make_problem("p3", pb.poisson3d(12))
        A = P.A
        lo = cgvk.partition_rows(A.n, world, 144)
        rp, ci, va = cgvk.local_rows(A, lo, rank)
        h = cgvk.halo_plan(A.n, lo, rank, rp, ci)
        loc, hb = cgvk.rank_local_columns(A.n, lo, rank, rp, ci)
        m = int(lo[rank + 1] - lo[rank])
        nl, nu = len(h["lower"]), len(h["upper"])
        # z-slabs: send rows are exactly a prefix and a suffix (peer-memory eligible)
        assert np.array_equal(h["send_lo"], np.arange(len(h["send_lo"])))
        assert np.array_equal(h["send_hi"], np.arange(m - len(h["send_hi"]), m))
        assert hb == ((m + 31) // 32 * 32 if nl + nu else m)
        x = P.x_star[lo[rank]:lo[rank + 1]]
        xloc = np.full(hb + nl + nu, np.nan)  # the pad is never read
        xloc[:m] = x
        sizes = torch.tensor([len(h["send_lo"]), len(h["send_hi"]), nl, nu], dtype=torch.int64)
        allsz = [torch.zeros(4, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(allsz, sizes)
        if rank > 0:  # the lower neighbour's suffix is my lower halo, and I am its upper halo
            assert int(allsz[rank - 1][1]) == nl and int(allsz[rank - 1][3]) == len(h["send_lo"])
        reqs = []
        if rank > 0:
            reqs.append(dist.isend(torch.from_numpy(x[h["send_lo"]].copy()), rank - 1))
            buf_lo = torch.zeros(nl, dtype=torch.float64)
            reqs.append(dist.irecv(buf_lo, rank - 1))
        if rank + 1 < world:
            reqs.append(dist.isend(torch.from_numpy(x[h["send_hi"]].copy()), rank + 1))
            buf_hi = torch.zeros(nu, dtype=torch.float64)
            reqs.append(dist.irecv(buf_hi, rank + 1))
        for rq in reqs:
            rq.wait()
        if rank > 0:
            xloc[hb:hb + nl] = buf_lo.numpy()
        if rank + 1 < world:
            xloc[hb + nl:] = buf_hi.numpy()
        y = OP.local_spmv(rp, loc, va, xloc)
        assert not np.isnan(y).any()  # no row read the pad
        part = O.dot(y, y, ("tree", 256, 1776, 0))
        parts = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, torch.tensor([part], dtype=torch.float64))
        tot = 0.0
        for t in parts:
            tot = tot + float(t.item())
        ys = [torch.zeros(int(lo[r + 1] - lo[r]), dtype=torch.float64) for r in range(world)]
        dist.all_gather(ys, torch.from_numpy(y))
        q.put((rank, np.concatenate([t.numpy() for t in ys]), tot))
    except BaseException as e:  # report instead of leaving the parent waiting
        q.put((rank, None, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_library_partition_halo_and_local_numbering(world):
    """world_size 2 / 3 gloo processes driving libcgvk's partition, halo plan
    and rank-local numbering: the distributed SpMV equals the global
    reference spmv bit-for-bit and the rank-ordered dot equals ORC_DOT_PART."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_lib, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, y, tot in res:
        assert y is not None, f"rank {rank}: {tot}"
    P = pb.make_problem("p3", pb.poisson3d(12))
    y_ref = O.spmv(P.A, P.x_star)
    lo = OP.partition_rows(P.A.n, world, 144)
    want = O.dot(y_ref, y_ref, ("part", 256, 1776, lo, 0))
    for rank, y, tot in res:
        assert np.array_equal(y.view(np.int64), y_ref.view(np.int64))
        assert tot == want


@pytest.mark.parametrize("nparts", [2, 3, 8])
def test_rank_local_numbering_matches_restatement(nparts):
    """cgvk_rank_local_columns == oracle/partition.py's [own | lower | upper]
    numbering with the halo moved to hbase (own rows rounded up to 32)."""
    A = pb.poisson3d(16)
    lo = cgvk.partition_rows(A.n, nparts, 256)
    for r in range(nparts):
        rp, ci, va = cgvk.local_rows(A, lo, r)
        loc, hb = cgvk.rank_local_columns(A.n, lo, r, rp, ci)
        _, want, _, _ = OP.local_matrix(A, lo, r)
        m = int(lo[r + 1] - lo[r])
        assert hb == (m + 31) // 32 * 32
        assert np.array_equal(np.where(want >= m, want - m + hb, want), loc)


def test_parallel_host_plan_matches_restatement_and_reports_first_error():
    """Shards above 2^20 entries take the threaded host path (halo plan and
    local numbering in row chunks): same maps as the restatement, and of
    several invalid rows the first one's error is reported, as a sequential
    scan would."""
    A = pb.poisson3d(80)  # 512,000 rows, 3.5 M entries: 1.75 M per rank at P = 2
    lo = cgvk.partition_rows(A.n, 2, 80 * 80)
    for r in range(2):
        rp, ci, va = cgvk.local_rows(A, lo, r)
        assert rp[-1] >= 1 << 20
        got = cgvk.halo_plan(A.n, lo, r, rp, ci)
        want = OP.halo_maps(A, lo, r)
        for k in ("lower", "upper", "send_lo", "send_hi"):
            assert np.array_equal(got[k], want[k]), (r, k)
        loc, hb = cgvk.rank_local_columns(A.n, lo, r, rp, ci)
        _, wloc, _, _ = OP.local_matrix(A, lo, r)
        m = int(lo[r + 1] - lo[r])
        assert np.array_equal(np.where(wloc >= m, wloc - m + hb, wloc), loc)
    rp, ci, va = cgvk.local_rows(A, lo, 0)
    bad = ci.copy()
    late, early = int(rp[200000]), int(rp[1000])
    bad[late] = A.n + 5                      # column out of range, late row
    bad[early], bad[early + 1] = bad[early + 1], bad[early]  # unsorted, early row
    with pytest.raises(cgvk.InvalidArgument, match="strictly increasing"):
        cgvk.halo_plan(A.n, lo, 0, rp, bad)
    bad[early], bad[early + 1] = bad[early + 1], bad[early]
    with pytest.raises(cgvk.InvalidArgument, match="out of range"):
        cgvk.halo_plan(A.n, lo, 0, rp, bad)
