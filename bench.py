#!/usr/bin/env python3
"""Benchmark: CG iterations/s and effective HBM GB/s per variant (BASELINE.json
metric) on the BASELINE.json configs[1] workload — 3D Poisson 7-point 128^3
(n=2,097,152, nnz=14,581,760), fp64 CSR, Jacobi, b = A x*, x* ~ U(-1,1) seeded,
x0 = 0 — for the six variants HS, CG-CG, M, PR, GV, pipe-PR.

A "step" is one CG iteration of each of the six variants (six solvers share
the matrix), so `value` = 6*K / (sum of the six device-timed K-iteration
runs) is the aggregate CG iterations/s; per-variant it/s, GB/s and roofline
fractions are in `per_variant`. Timing: CUDA events on each solver's stream
around K graph-replayed iterations (inputs resident in HBM; the per-iteration
working set, 368-536 MB, exceeds the 126 MB L2, so no flush is needed).

`e2e` goes through the public C ABI with pinned host buffers: matrix upload
(int64 CSR, validated and narrowed on the device), then per variant
cgvk_solve(K iterations) including the b/x0 upload and the x download.

--impl reference times the reference's own CPU solver (oracle/_ref, the
unchanged reference sources; the C restatement if that library is absent) on
the host cores: the six variants in six threads, K steps each.

Multi-GPU (torchrun, N>1): the same global solve row-partitioned into z-slabs
(one rank per GPU, NCCL halo exchange + rank-ordered reductions; "scaling":
"strong"); each variant's K iterations are device-timed on every rank and the
max over ranks is taken. --emulate-ranks P runs the partitioned data path with
P in-process ranks on one GPU.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

VARIANTS = ["hs", "cg", "m", "pr", "gv", "pipe-pr"]
# Algorithmic vector traffic per kernel launch (n-length fp64 vectors), Jacobi
# / none: (update kernel K1, SpMV kernel K2); K2 additionally streams A once.
# Iteration totals are SURVEY App. A's minimum V (HS 11, CG 13, M/PR 15, GV 21,
# pipe 19). HS stores r~ in K1 and gathers it in K2 (same total as App. A's
# split 4+7); CG and GV also store their gathered r~ / w~ (one extra write
# each) — counted as overhead, not work.
KERNEL_VECTORS = {
    "hs": {True: (5, 6), False: (3, 6)},
    "cg": {True: (10, 3), False: (8, 3)},
    "m": {True: (10, 5), False: (6, 4)},
    "pr": {True: (10, 5), False: (6, 4)},
    "gv": {True: (18, 3), False: (13, 2)},
    "pipe-pr": {True: (15, 4), False: (11, 3)},
    "pipe-pr-m": {True: (15, 4), False: (11, 3)},
}
KERNEL_NAMES = {"hs": ("hs_k1", "hs_k2"), "cg": ("cg_k1", "cg_k2"), "m": ("pr_k1", "pr_k2"),
                "pr": ("pr_k1", "pr_k2"), "gv": ("gv_k1", "gv_k2"),
                "pipe-pr": ("ppr_k1", "ppr_k2"), "pipe-pr-m": ("ppr_k1", "ppr_k2")}


def a_bytes(n: int, nnz: int) -> int:
    return 12 * nnz + 4 * (n + 1)


def iter_bytes(v: str, n: int, nnz: int, prec: bool) -> int:
    k1, k2 = KERNEL_VECTORS[v][prec]
    return a_bytes(n, nnz) + 8 * n * (k1 + k2)


def peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured"}
    return {"hbm_gbs": 6650.0, "source": "fallback"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (FileNotFoundError, OSError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.perf_counter(), line.strip()))

    def wait_first(self, timeout: float = 5.0) -> None:
        t0 = time.perf_counter()
        while self.proc and not self.lines and time.perf_counter() - t0 < timeout:
            time.sleep(0.01)

    def mark(self, name: str) -> None:
        setattr(self, name, time.perf_counter())

    def stop(self) -> dict | None:
        if not self.proc:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        t0, t1 = getattr(self, "t_start", None), getattr(self, "t_end", None)
        lines = [ln for ts, ln in self.lines if t0 is None or t0 <= ts <= t1 + 0.025]
        in_region = len(lines)
        if not lines:  # region shorter than the sampling period: nearest samples
            lines = [ln for _, ln in self.lines[-3:]]
        for ln in lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for name, val in zip(names, f[4:8]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "samples_in_timed_region": in_region}


def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("gloo")
        return rank, local, world, dist
    return rank, local, world, None


def max_over_ranks(dist, value: float) -> float:
    if dist is None:
        return value
    import torch

    t = torch.tensor([value], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(dist):
    if dist is not None:
        dist.barrier()


# ------------------------------------------------------------------ CPU arms
#
# Nothing below maps a library of the product package: variant ids come from
# this table (inc/variants.hpp:17-25, the reference's enum order) and the
# inputs from oracle/_build/libinputgen.so (a second build of the App. B
# generator source), so the reference arm's process loads only oracle/.

VARIANT_IDS = {"hs": 0, "cg": 1, "m": 2, "pr": 3, "gv": 4, "pipe-pr-m": 5, "pipe-pr": 6}
INPUTGEN = os.path.join(ROOT, "oracle", "_build", "libinputgen.so")
# bounded single-core samples (BASELINE.md §3 asks K = 50 for the Poisson
# configs, best of 3; the two largest configs take ~0.3-0.5 s per step on one
# core, so their sample is K = 5, best of 2, to keep the run within minutes)
CPU_SAMPLE = {"p2d": (50, 3), "p64": (50, 3), "p128": (50, 3), "v256": (5, 2), "r4m": (5, 2)}


def host_problem(name: str):
    """App. B inputs built by the oracle's copy of the generators."""
    from paper_1905_01549_b200 import problems as pb

    if os.path.exists(INPUTGEN) and pb._gen is None:
        pb.use_generator(INPUTGEN)
    return pb.config_problem(name)


def host_info() -> dict:
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                model = ln.split(":", 1)[1].strip()
    except (OSError, subprocess.SubprocessError):
        pass
    return {"nproc": os.cpu_count(), "affinity": len(os.sched_getaffinity(0)), "lscpu_model": model}


def cpu_sweep(P, variants, steps: int, warmup: int, kind: str):
    """The six variants in six threads (the reference's jobs>1 model,
    src/experiment.cpp:317-322); each thread runs `steps` step() calls."""
    from oracle import oracle as O

    solvers = []
    for v in variants:
        vid = VARIANT_IDS[v]
        if kind == "reference":
            solvers.append(O.Reference(P.A, vid, 1, P.b, P.x0))
        else:
            solvers.append(O.Restatement(P.A, vid, 1, P.b, P.x0))
    if warmup:
        ths = [threading.Thread(target=s.time_steps, args=(warmup,)) for s in solvers]
        [t.start() for t in ths]
        [t.join() for t in ths]
    res = [None] * len(solvers)

    def work(i):
        res[i] = solvers[i].time_steps(steps)

    ths = [threading.Thread(target=work, args=(i,)) for i in range(len(solvers))]
    t0 = time.perf_counter()
    [t.start() for t in ths]
    [t.join() for t in ths]
    wall = time.perf_counter() - t0
    iters = sum(r[1] for r in res)
    per = {v: {"it_per_s": r[1] / r[0] if r[0] > 0 else None, "ms_per_iter": 1e3 * r[0] / max(r[1], 1)}
           for v, r in zip(variants, res)}
    return iters, wall, per


def cpu_worker(args) -> int:
    """(run under taskset by single_core_baseline) the reference's step() loop
    on one core: per variant one warm-up step, then the best of `reps` timed
    runs of `steps` step() calls (std::chrono inside oracle/ref_shim.cpp)."""
    from oracle import oracle as O

    P = host_problem(args.cpu_worker)
    kind = "reference" if O.reference_available() else "port"
    mat = O.RefMatrix(P.A) if kind == "reference" else None
    steps, reps = args.cpu_steps, args.cpu_reps
    out = {}
    for v in VARIANTS:
        if kind == "reference":
            s = O.Reference(P.A, VARIANT_IDS[v], 1, P.b, P.x0, mat=mat)
        else:
            s = O.Restatement(P.A, VARIANT_IDS[v], 1, P.b, P.x0)
        s.time_steps(1)
        best = None
        for _ in range(reps):
            secs, it = s.time_steps(steps)
            ms = 1e3 * secs / max(it, 1)
            best = ms if best is None else min(best, ms)
        out[v] = best
        del s
    print(json.dumps({"kind": kind, "ms_per_iter": out, "steps": steps, "reps": reps,
                      "affinity": sorted(os.sched_getaffinity(0))}), flush=True)
    return 0


def single_core_baseline(cfg: str, steps: int | None = None, reps: int | None = None) -> dict | None:
    """The baseline of record: the reference's step() on ONE
    pinned core (taskset), best of `reps` runs of K steps per variant."""
    k, r = CPU_SAMPLE[cfg]
    steps, reps = steps or k, reps or r
    core = sorted(os.sched_getaffinity(0))[-1]
    cmd = ["taskset", "-c", str(core), sys.executable, os.path.abspath(__file__), "--cpu-worker", cfg,
           "--cpu-steps", str(steps), "--cpu-reps", str(reps)]
    t0 = time.perf_counter()
    try:
        r_ = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
        d = json.loads(r_.stdout.strip().splitlines()[-1])
    except (OSError, subprocess.SubprocessError, ValueError, IndexError) as e:
        return {"error": f"{type(e).__name__}: {e}"}
    ms = d["ms_per_iter"]
    total = sum(ms.values())
    return {"value": len(ms) / (total * 1e-3), "unit": "iterations/s", "cores": 1, "kind": d["kind"],
            "pinned_core": core,
            "sample": f"{steps} step() calls per variant, best of {reps}, one after another on one "
                      f"core pinned with taskset (value = 6 / sum of the six ms/iteration)",
            "ms_per_iter": ms, "wall_s": round(time.perf_counter() - t0, 1), "host": host_info()}


def run_reference_arm(args, rank, world, dist):
    if rank != 0:
        return 0
    from oracle import oracle as O

    kind = "reference" if O.reference_available() else "port"
    P = host_problem(args.config)
    iters, wall, per = cpu_sweep(P, VARIANTS, args.steps, args.warmup, kind)
    value = iters / wall
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "iterations/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * wall / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args.config, P),
        "cpu_baseline": {"value": value, "unit": "iterations/s", "cores": len(VARIANTS),
                         "kind": kind,
                         "sample": f"{args.steps} step() calls of each of the six variants on "
                                   f"{args.config}, one thread per variant (oracle/_ref: the "
                                   f"unchanged reference sources)",
                         "host": host_info()},
        "e2e": {"value": value, "unit": "iterations/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "per_variant": per,
    }
    print(json.dumps(line), flush=True)
    return 0


METRIC = "CG iterations/s (six-variant sweep) and effective HBM GB/s per variant"


def workload_config(name, P, ranks: int = 1) -> dict:
    per = [iter_bytes(v, P.A.n, P.A.nnz, True) / max(ranks, 1) / 1e6 for v in VARIANTS]
    lo, hi = min(per), max(per)
    l2 = (f"per-GPU working set {lo:.0f}-{hi:.0f} MB per iteration > L2 (126 MB); no flush needed"
          if lo > 126 else
          f"per-GPU working set {lo:.0f}-{hi:.0f} MB per iteration fits the 126 MB L2: the solve runs "
          f"L2-resident as it would in use (latency-bound regime, SURVEY 8d); no flush")
    return {"workload": f"{name} ({P.A.n} rows, {P.A.nnz} nnz) fp64 CSR, Jacobi, "
                        f"six variants, K fixed iterations each",
            "variants": VARIANTS, "n": P.A.n, "nnz": P.A.nnz, "precond": "jacobi",
            "l2": l2, "parallelism": "single-gpu"}


# ------------------------------------------------------------------ GPU arm

def load_traffic() -> dict:
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return {}


ALIGN = {"p2d": 256, "p64": 64 * 64, "p128": 128 * 128, "v256": 256 * 256, "r4m": 1}


_COMMS = {}  # communicators of this process, by (kind, ranks / world, rank, device)


class SolveSet:
    """One solver per variant: single-GPU, one NCCL rank of a row-partitioned
    solve (torchrun, one process per GPU), or P in-process ranks on one GPU
    (--emulate-ranks, the partitioned data path without NCCL)."""

    def __init__(self, args, P, rank, world, device, dist, pinned=None, replicas=False, on_solver=None,
                 p2p=False, variants=None):
        from paper_1905_01549_b200 import cgvk
        from paper_1905_01549_b200.cgvk import Precond, VariantConfig, variant_from_name

        A = P.A
        rp, ci, va, b, x0 = pinned or (A.row_ptr, A.col_idx, A.values, P.b, P.x0)
        self.groups, self.solvers, self.comm, self.mats = [], {}, None, []
        variants = variants or VARIANTS
        cfgs = {v: VariantConfig.make(variant_from_name(v)) for v in variants}
        self.transport = None
        ranks = world if world > 1 else args.emulate_ranks
        if replicas or (ranks <= 1 and not args.nccl):
            t = time.perf_counter()
            self.mats = [cgvk.DeviceMatrix(A.n, rp, ci, va, device=device)]
            self.t_matrix = time.perf_counter() - t
            for v in variants:
                self.solvers[v] = cgvk.initialize(cfgs[v], self.mats[0], Precond.JACOBI, b, x0)
                if on_solver:  # the user's next calls on it (e2e: step, x download), enqueued at once
                    on_solver(v, self.solvers[v])
            self.t_init = time.perf_counter() - t - self.t_matrix
            return
        ranks = max(ranks, 1)
        if os.environ.get("CGVK_BENCH_FAIL_PARTITION"):  # exercises the replica fallback
            raise RuntimeError("CGVK_BENCH_FAIL_PARTITION set")
        lo = cgvk.partition_rows(A.n, ranks, ALIGN[args.config])
        Acsr = type(A)(A.n, rp, ci, va)
        # the communicator is process set-up (like the CUDA context): created
        # once, shared by every solve of the run, outside the timed regions
        if world > 1 or args.nccl:  # NCCL: this process drives rank `rank`
            key = ("nccl", world, rank, device)
            if key not in _COMMS:
                nid = cgvk.nccl_unique_id() if rank == 0 else None
                obj = [nid]
                if dist is not None:
                    dist.broadcast_object_list(obj, src=0)
                _COMMS[key] = cgvk.Comm(world, rank, device, obj[0])
            mine = [rank]
        else:
            key = ("local", ranks, device)
            if key not in _COMMS:
                _COMMS[key] = cgvk.Comm(ranks, 0, device)
            mine = list(range(ranks))
        self.comm = _COMMS[key]
        self.mats = [cgvk.RankMatrix(A.n, lo, r, *cgvk.local_rows(Acsr, lo, r), device=device) for r in mine]
        for v in variants:
            g = cgvk.Group(self.comm, self.mats, cfgs[v], Precond.JACOBI,
                           [b[lo[r]:lo[r + 1]] for r in mine], [x0[lo[r]:lo[r + 1]] for r in mine],
                           p2p=p2p)
            self.transport = g.transport
            self.groups.append(g)
            self.solvers[v] = g.solvers[0]  # time_steps on member 0 steps the whole local group

    def close(self):
        for g in self.groups:
            g.close()
        for s in self.solvers.values():
            s.close()
        for m in self.mats:
            m.close()


def p2p_self_check(args, P, rank, world, device, dist, iters: int = 12) -> None:
    """The peer-memory transport must reproduce the copy / NCCL exchange bit
    for bit (residual histories of HS and pipe-PR, 12 iterations) before it
    is timed; raises otherwise (bench falls back to the copy exchange)."""
    hist = {}
    fail = None
    for p2p in (True, False):
        # group creation is collective (a failed set-up fails on every rank);
        # a rank whose solve gives up keeps taking part, and the verdict is
        # agreed over the ranks before anyone moves on
        S = SolveSet(args, P, rank, world, device, dist, p2p=p2p, variants=["hs", "pipe-pr"])
        try:
            if p2p and S.transport != "p2p":
                fail = fail or f"peer-memory transport not selected ({S.transport})"
            for v, s in S.solvers.items():
                s.step(iters)
                try:
                    s.sync()
                    hist[(p2p, v)] = s.history()
                except Exception as e:  # noqa: BLE001
                    fail = fail or f"{v}: {type(e).__name__}: {e}"
        finally:
            S.close()
    ok = 0.0 if fail else 1.0
    if dist is not None:
        ok = -max_over_ranks(dist, -ok)
    if ok < 1.0:
        raise RuntimeError(fail or "peer-memory self-check failed on another rank")
    for v in ("hs", "pipe-pr"):
        a, b = hist[(True, v)], hist[(False, v)]
        if a.shape != b.shape or not np.array_equal(a.view(np.int64), b.view(np.int64)):
            raise RuntimeError(f"peer-memory self-check: {v} history differs from the copy exchange")


def measure_config(args, cfg_name, rank, local, world, dist, extra=False) -> dict:
    """Device-timed sweep, per-kernel shares, roofline and e2e of one config."""
    from paper_1905_01549_b200 import cgvk, problems as pb
    from paper_1905_01549_b200.cgvk import Precond, VariantConfig, variant_from_name

    device = local
    args = argparse.Namespace(**{**vars(args), "config": cfg_name})
    P = pb.config_problem(cfg_name)
    n, nnz = P.A.n, P.A.nnz
    pk = peaks()
    partitioned = not extra and (world > 1 or args.emulate_ranks > 1 or args.nccl)
    fallback = None
    S = None
    notes = []
    # row-partitioned transports, best first: peer memory (in-kernel, after a
    # bit-for-bit self-check against the copy / NCCL exchange), then copy /
    # NCCL; every rank takes the same one
    ladder = ["p2p", "copy"] if args.transport == "auto" else [args.transport]
    for tr in ladder if partitioned else ["single"]:
        try:
            if S is not None:
                S.close()
                S = None
            if tr == "p2p":
                p2p_self_check(args, P, rank, world, device, dist)
            S = SolveSet(args, P, rank, world, device, dist, replicas=extra, p2p=tr == "p2p")
            for v, s in S.solvers.items():  # warm-up: graphs, clocks, caches
                s.time_steps(args.warmup)
                s.sync()
            ok = 1.0
        except Exception as e:  # noqa: BLE001 — reported in the JSON line
            if not partitioned:
                raise
            ok = 0.0
            notes.append(f"{tr}: {type(e).__name__}: {e}")
        if partitioned and dist is not None:
            ok = -max_over_ranks(dist, -ok)  # min over ranks: every rank moves on together
        if ok >= 1.0:
            break
    tnotes = "; ".join(notes) if notes else None
    if partitioned and ok < 1.0:
        fallback = tnotes
        # the row-partitioned transport failed on this box: independent
        # replicas (weak scaling), labelled as such in `parallelism`
        if S is not None:
            S.close()
        fallback = fallback or "another rank's partitioned setup failed"
        partitioned = False
        S = SolveSet(args, P, rank, world, device, dist, replicas=True)
        for v, s in S.solvers.items():
            s.time_steps(args.warmup)

    clocks = ClockSampler(device) if not args.no_clocks else None
    if clocks:
        clocks.start()
        clocks.wait_first()
    barrier(dist)
    if clocks:
        clocks.mark("t_start")
    per = {}
    total_ms, total_iters = 0.0, 0
    for v, s in S.solvers.items():
        barrier(dist)
        ms, it = s.time_steps(args.steps)
        ms = max_over_ranks(dist, ms)
        per[v] = {"ms": ms, "iters": it, "launches_per_iter": s.launches_per_iter(),
                  "launches": s.launches(args.steps)}
        total_ms += ms
        total_iters += it
    if clocks:
        clocks.mark("t_end")
        time.sleep(0.05)
    clk = clocks.stop() if clocks else None
    barrier(dist)
    S.close()

    # per-kernel device times (events around each launch, same stream); the
    # partitioned path interleaves exchanges, so only the single-GPU run has it
    kernels = []
    if not partitioned:
        A = cgvk.DeviceMatrix.from_csr(P.A, device=device)
        prof_iters = min(args.steps, 20)
        for v in VARIANTS:
            s = cgvk.initialize(VariantConfig.make(variant_from_name(v)), A, Precond.JACOBI, P.b, P.x0)
            s.time_steps(2)
            k1, k2, it = s.profile(prof_iters)
            names = KERNEL_NAMES[v]
            vec = KERNEL_VECTORS[v][True]
            b1 = 8 * n * vec[0]
            b2 = a_bytes(n, nnz) + 8 * n * vec[1]
            # An event between two launches breaks the programmatic-dependent
            # overlap and the chained schedule the graph runs with, so the
            # event-timed launches sum to more than the graph's iteration
            # (P128 GV: 108 vs 93 us). Each kernel's time in the timed region
            # = the graph iteration time (events, above) x its share of the
            # event-timed pair; the raw per-launch times are kept.
            t_it = per[v]["ms"] / max(per[v]["iters"], 1)
            f1 = k1 / (k1 + k2) if k1 + k2 > 0 else 0.5
            rows = ((names[0], b1, k1 / it, f1), (names[1], b2, k2 / it, 1.0 - f1))
            if s.launches_per_iter() == 1:  # one kernel per iteration (PR / M on an L2-resident problem)
                rows = ((names[0].replace("_k1", "_f"), b1 + b2, k1 / it, 1.0),)
            for name, b, raw, f in rows:
                ms = t_it * f
                kernels.append({"variant": v, "kernel": name, "ms_per_launch": ms,
                                "ms_per_launch_unfused": raw, "bytes_per_launch": b,
                                "gbs": b / (ms * 1e-3) / 1e9})
            s.close()
        A.close()

    reps = world if (fallback is not None or extra) and world > 1 else 1
    for v in VARIANTS:
        d = per[v]
        t_iter = d["ms"] / max(d["iters"], 1) * 1e-3
        bi = iter_bytes(v, n, nnz, True) * reps  # every replica moves the whole iteration's bytes
        per[v].update({"it_per_s": reps * d["iters"] / (d["ms"] * 1e-3), "us_per_iter": t_iter * 1e6,
                       "bytes_per_iter": bi, "gbs": bi / t_iter / 1e9,
                       "roofline_frac": bi / t_iter / 1e9 / (pk["hbm_gbs"] * max(world, 1)),
                       "roofline_frac_nominal_8tbs": bi / t_iter / 1e9 / (8000.0 * max(world, 1))})
    traffic = load_traffic().get(cfg_name, {})
    if kernels:
        top = max(kernels, key=lambda k: k["ms_per_launch"])
        roof = {"bound": "hbm", "kernel": top["kernel"], "variant": top["variant"],
                "achieved": top["gbs"], "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": top["gbs"] / pk["hbm_gbs"], "peak_source": pk["source"],
                "traffic": traffic.get(top["kernel"]),
                "bytes_per_launch": top["bytes_per_launch"], "ms_per_launch": top["ms_per_launch"],
                "timing": "kernel share of the event-timed K1/K2 launches x the event-timed graph "
                          "iteration; ms_per_launch_unfused in `kernels`"}
        for k in kernels:  # ncu DRAM bytes beside the algorithmic bytes (K1s re-read K2's output from L2)
            if k["kernel"] in traffic:
                k["dram_bytes_ncu"] = traffic[k["kernel"]]
    else:  # partitioned: whole-iteration roofline of the slowest variant over all GPUs
        worst = min(VARIANTS, key=lambda v: per[v]["roofline_frac"])
        roof = {"bound": "hbm", "kernel": "iteration", "variant": worst,
                "achieved": per[worst]["gbs"], "peak": pk["hbm_gbs"] * world, "unit": "GB/s",
                "frac": per[worst]["roofline_frac"], "peak_source": pk["source"], "traffic": None,
                "bytes_per_launch": per[worst]["bytes_per_iter"],
                "ms_per_launch": per[worst]["us_per_iter"] * 1e-3}
    iteration_frac = {v: round(per[v]["roofline_frac"], 4) for v in VARIANTS}

    e2e = None if args.no_e2e else measure_e2e(args, P, rank, world, device, dist,
                                                replicas=fallback is not None or extra,
                                                p2p=S.transport == "p2p")

    value = reps * total_iters / (total_ms * 1e-3)
    cfg = workload_config(cfg_name, P, world if partitioned else 1)
    if partitioned:
        p2p = S.transport == "p2p"
        via = "peer memory: in-kernel stamped stores" if p2p else "NCCL"
        cfg["parallelism"] = (f"row-partitioned z-slabs over {world} GPUs ({via})" if world > 1 or args.nccl
                              else f"row-partitioned, {args.emulate_ranks} in-process ranks on 1 GPU"
                                   + (" (peer-memory exchange)" if p2p else " (copy exchange)"))
        cfg["transport"] = S.transport
        if tnotes:
            cfg["transport_notes"] = tnotes
    if fallback is not None:
        cfg["parallelism"] = f"{world} independent replicas (row-partitioned transport failed: {fallback})"
    elif extra and world > 1:
        cfg["parallelism"] = f"{world} independent replicas"
    # our kernels in the timed region: one limit-setting launch per step()
    # call + the captured kernels of every replayed graph (chained graphs'
    # tail kernel, halo pack/unpack and finalize kernels included; NCCL's
    # own not counted)
    launches = sum(per[v]["launches"] for v in VARIANTS)
    return {"value": value, "ms_per_step": total_ms / args.steps, "config": cfg, "roofline": roof,
            "iteration_roofline_frac": iteration_frac, "kernels": kernels, "per_variant": per,
            "gpu_launches": launches * world, "e2e": e2e, "clocks": clk,
            "scaling": "weak" if reps > 1 else "strong"}


def measure_e2e(args, P, rank, world, device, dist, replicas=False, p2p=False) -> dict:
    """e2e through the public API with pinned host buffers."""
    from paper_1905_01549_b200 import cgvk

    n = P.A.n
    arrs = [P.A.row_ptr.copy(), P.A.col_idx.copy(), P.A.values.copy(), P.b.copy(), P.x0.copy()]
    xs = {v: np.empty(n) for v in VARIANTS}  # the user's result buffers (registered, like the inputs)
    for arr in arrs + list(xs.values()):
        cgvk.host_register(arr)

    def sweep():
        # the user's calls: upload A (validated on the device: synchronous),
        # then per variant create a solver (b, x0 up; initialize() stream-
        # ordered), step it K times and enqueue the x download into the
        # user's registered buffer; then wait for all. Every solver runs on its
        # own stream, so uploads, solves and downloads of different solvers
        # overlap
        ph = {}
        t = time.perf_counter()
        prev = []

        def on_solver(v, s):
            if args.e2e_order == "chained" and prev:
                # this solve's iterations start after the previous solve's
                # (their kernels do not interleave on the SMs); its upload
                # (already enqueued) and the previous download still overlap
                pv, ps = prev[-1]
                s.after(ps)
                ps.x_async(xs[pv])
                s.step(args.steps)
            elif args.e2e_order == "chained":
                s.step(args.steps)
            else:
                s.step(args.steps)
                s.x_async(xs[v])
            prev.append((v, s))

        E = SolveSet(args, P, rank, world, device, dist, pinned=tuple(arrs), replicas=replicas, p2p=p2p,
                     on_solver=on_solver)
        if args.e2e_order == "chained" and prev:
            prev[-1][1].x_async(xs[prev[-1][0]])
        ph["enqueue_ms"] = 1e3 * (time.perf_counter() - t)
        if hasattr(E, "t_matrix"):
            ph["matrix_upload_ms"] = 1e3 * E.t_matrix
        its = 0
        xx = None
        for v, s in E.solvers.items():
            if E.groups:  # a rank of a row-partitioned group
                s.step(args.steps)
            s.sync()
            xx = xs[v] if not E.groups else s.x
            its += s.k
        ph["until_done_ms"] = 1e3 * (time.perf_counter() - t)
        return its, xx, ph, E

    try:
        barrier(dist)
        sweep()[3].close()  # warm-up sweep (driver/allocator state, pinned mappings)
        # best of --e2e-reps timed sweeps (each max over ranks), as the
        # paper reports minima over repetitions: one host
        # hiccup must not stand for the path
        wall = None
        for _ in range(max(args.e2e_reps, 1)):
            barrier(dist)
            t0 = time.perf_counter()
            its_r, x_r, ph_r, E = sweep()
            t1 = time.perf_counter()
            E.close()  # freeing device memory is not part of the user's solve
            barrier(dist)
            w = max_over_ranks(dist, t1 - t0)
            if wall is None or w < wall:
                wall, e2e_iters, x, phases = w, its_r, x_r, ph_r
    finally:
        for arr in arrs + list(xs.values()):
            cgvk.host_unregister(arr)
    reps = world if replicas and world > 1 else 1
    h2d = sum(a.nbytes for a in arrs[:3]) + len(VARIANTS) * (arrs[3].nbytes + arrs[4].nbytes)
    d2h = len(VARIANTS) * x.nbytes
    return {"value": reps * e2e_iters / wall, "unit": "iterations/s",
            "h2d_bytes_per_step": h2d // args.steps, "d2h_bytes_per_step": d2h // args.steps,
            "phases_ms": {k: round(v, 2) for k, v in phases.items()}, "order": args.e2e_order,
            "note": "fastest of --e2e-reps timed sweeps after one warm-up sweep: int64 CSR + b, x0 per variant up "
                    "(each rank its rows), K steps, x per variant down, all inside the timed region; "
                    "bytes_per_step = sweep bytes / K (rank 0's share when N > 1)"}


def run_gpu_arm(args, rank, local, world, dist):
    head = measure_config(args, args.config, rank, local, world, dist)
    extras = {}
    if world == 1 and args.emulate_ranks <= 1 and not args.nccl:
        for c in [c for c in args.per_config.split(",") if c and c != args.config]:
            extras[c] = measure_config(args, c, rank, local, world, dist, extra=True)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        from oracle import oracle as O

        kind = "reference" if O.reference_available() else "port"
        P = host_problem(args.config)
        iters, wall, cper = cpu_sweep(P, VARIANTS, args.cpu_steps, 1, kind)
        del P
        cpu = {"value": iters / wall, "unit": "iterations/s", "cores": len(VARIANTS), "kind": kind,
               "sample": f"{args.cpu_steps} step() calls of each of the six variants on {args.config} "
                         f"(one thread per variant, the reference's own -O2 -ffp-contract=off build)",
               "per_variant": cper,
               "single_core": None if args.no_single_core else single_core_baseline(args.config)}
        for c, d in extras.items():
            d["cpu_baseline"] = None if args.no_single_core else single_core_baseline(c)

    if rank == 0:
        line = {
            "metric": METRIC, "value": head["value"], "unit": "iterations/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": head["ms_per_step"],
            "higher_is_better": True, "scaling": head["scaling"], "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (App. B generator, x* from mt19937_64(1))",
            "config": head["config"],
            "roofline": head["roofline"],
            "iteration_roofline_frac": head["iteration_roofline_frac"],
            "kernels": head["kernels"],
            "per_variant": head["per_variant"],
            "gpu_launches": head["gpu_launches"] + sum(d["gpu_launches"] for d in extras.values()),
            "e2e": head["e2e"],
            "cpu_baseline": cpu,
            "clocks": head["clocks"],
        }
        if extras:
            line["per_config"] = {c: {k: d[k] for k in ("value", "ms_per_step", "config", "roofline",
                                                         "iteration_roofline_frac", "per_variant", "kernels",
                                                         "gpu_launches", "e2e", "clocks", "cpu_baseline")
                                      if k in d} for c, d in extras.items()}
        print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=os.environ.get("BENCH_CONFIG", "p128"), choices=["p2d", "p64", "p128", "v256", "r4m"])
    ap.add_argument("--per-config", default=os.environ.get("BENCH_PER_CONFIG", "v256,r4m,p64,p2d"),
                    help="further single-GPU configs measured after the headline one (own roofline, e2e, "
                         "clocks, single-core CPU baseline each); '' for none")
    ap.add_argument("--cpu-steps", type=int, default=10)
    ap.add_argument("--cpu-reps", type=int, default=3)
    ap.add_argument("--cpu-worker", default=None, help=argparse.SUPPRESS)
    ap.add_argument("--no-clocks", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-reps", type=int, default=2, help="timed end-to-end sweeps; the fastest is reported")
    ap.add_argument("--e2e-order", default="chained", choices=["chained", "concurrent"],
                    help="e2e: each solve's iterations after the previous solve's (cgvk_solver_after), or all at once")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-single-core", action="store_true")
    ap.add_argument("--nccl", action="store_true",
                    help="row-partitioned path over NCCL even at one rank (transport check)")
    ap.add_argument("--transport", default="auto", choices=["auto", "p2p", "copy"],
                    help="row-partitioned solves: peer memory inside the kernels (CGVK_GROUP_P2P, after a "
                         "bit-exact self-check), the copy / NCCL exchange, or auto (p2p, else copy)")
    ap.add_argument("--emulate-ranks", type=int, default=1,
                    help="row-partitioned solve with P in-process ranks on one GPU")
    args = ap.parse_args()
    if args.cpu_worker:
        return cpu_worker(args)
    if args.warmup < 3:
        args.warmup = 3  # timing rule: at least 3 warm-up steps
    rank, local, world, dist = dist_init()
    try:
        if args.impl == "reference":
            return run_reference_arm(args, rank, world, dist)
        return run_gpu_arm(args, rank, local, world, dist)
    finally:
        if dist is not None:
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
