"""The reference's cost model (proj/include/cgvariants/cost_model.hpp,
proj/src/cost_model.cpp) and its calibration on a B200.

The model itself is host arithmetic, restated here with the same names,
formulas and argument checks; `calibrate()` measures its parameters with the
device (cgvk_time_ops: CUDA-event-timed SpMV, block SpMV and a global
reduction) so `iteration_time` can be set against the measured per-variant
iteration times of the fused kernels (scripts/cost_model.py).
"""
from __future__ import annotations

from dataclasses import dataclass, field

from .cgvk import Variant


@dataclass
class CostParams:
    """CostParams (cost_model.hpp:11-20); seconds (any consistent unit)."""
    c_gr: float = 0.0   # global reduction communication time
    t_mv: float = 0.0   # matrix-vector computation time
    c_mv: float = 0.0   # matrix-vector communication time
    t_2mv: float = 0.0  # fused two-product computation time

    def validate(self) -> None:  # src/cost_model.cpp:8-13
        if self.c_gr < 0.0 or self.t_mv < 0.0 or self.c_mv < 0.0 or self.t_2mv < 0.0:
            raise ValueError("cost parameters must be nonnegative")
        if self.t_mv > self.t_2mv or self.t_2mv > 2.0 * self.t_mv:
            raise ValueError("need t_mv <= t_2mv <= 2*t_mv")


def iteration_time(v: Variant, p: CostParams) -> float:
    """src/cost_model.cpp:15-30 (vector updates and local dots ignored)."""
    v = Variant(v)
    if v == Variant.HS:
        return 2.0 * p.c_gr + p.t_mv + p.c_mv
    if v in (Variant.CG_CG, Variant.M, Variant.PR):
        return p.c_gr + p.t_mv + p.c_mv
    if v == Variant.GV:
        return max(p.c_gr, p.t_mv + p.c_mv)
    return max(p.c_gr, p.t_2mv + p.c_mv)  # PIPE_PR_M, PIPE_PR


@dataclass
class ScalingScenario:
    nodes: list = field(default_factory=list)   # strictly increasing
    params: list = field(default_factory=list)  # one CostParams per node count


@dataclass
class ScalingPoint:
    nodes: int
    seconds: float


def _check_scenario(s: ScalingScenario) -> None:  # src/cost_model.cpp:34-44
    if not s.nodes:
        raise ValueError("empty scaling scenario")
    if len(s.nodes) != len(s.params):
        raise ValueError("scenario node and parameter counts differ")
    for a, b in zip(s.nodes, s.nodes[1:]):
        if b <= a:
            raise ValueError("node counts must be strictly increasing")
    for p in s.params:
        p.validate()


def predict_scaling(v: Variant, s: ScalingScenario, iterations: int = 1500) -> list:
    """src/cost_model.cpp:48-57."""
    _check_scenario(s)
    if iterations < 1:
        raise ValueError("iterations must be >= 1")
    return [ScalingPoint(n, float(iterations) * iteration_time(v, p)) for n, p in zip(s.nodes, s.params)]


def crossover_nodes(candidate: Variant, baseline: Variant, s: ScalingScenario):
    """src/cost_model.cpp:59-67: first node count where candidate is strictly faster."""
    _check_scenario(s)
    for n, p in zip(s.nodes, s.params):
        if iteration_time(candidate, p) < iteration_time(baseline, p):
            return n
    return None


def calibrate(A, reps: int = 50) -> tuple[CostParams, dict]:
    """Device-measured parameters for one GPU: t_mv = y = A x, t_2mv = the
    one-pass (A x1, A x2), c_gr = one global reduction (dot + last-CTA fold;
    on one GPU its cost is the grid-wide fold, not a network), c_mv = 0 (no
    halo on one GPU). t_2mv is clamped into [t_mv, 2 t_mv] as validate()
    requires. Returns (params in seconds, raw ms)."""
    ms = A.time_ops(reps)
    t_mv = ms["spmv"] * 1e-3
    t_2mv = min(max(ms["block_spmv"] * 1e-3, t_mv), 2.0 * t_mv)
    p = CostParams(c_gr=ms["dot"] * 1e-3, t_mv=t_mv, c_mv=0.0, t_2mv=t_2mv)
    p.validate()
    return p, ms
