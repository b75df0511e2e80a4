"""Cost model (proj/src/cost_model.cpp) restated in paper_1905_01549_b200/cost_model.py:
the reference's own test cases (proj/tests/test_cost_model.cpp), CPU only;
plus the device calibration on the GPU."""
import random

import pytest

from paper_1905_01549_b200 import cgvk, problems as pb
from paper_1905_01549_b200.cgvk import Variant
from paper_1905_01549_b200.cost_model import (CostParams, ScalingScenario, calibrate, crossover_nodes,
                                              iteration_time, predict_scaling)

ALL = list(Variant)


def expected(v, c_gr, t_mv, c_mv, t_2mv):  # independently hand-coded, as the reference test
    if v == Variant.HS:
        return c_gr + c_gr + t_mv + c_mv
    if v in (Variant.CG_CG, Variant.M, Variant.PR):
        return c_gr + t_mv + c_mv
    if v == Variant.GV:
        return c_gr if c_gr > t_mv + c_mv else t_mv + c_mv
    return c_gr if c_gr > t_2mv + c_mv else t_2mv + c_mv


def test_published_reference_point():
    p = CostParams(c_gr=1.0, t_mv=1.0, c_mv=0.0, t_2mv=1.5)
    want = {Variant.HS: 3.0, Variant.CG_CG: 2.0, Variant.M: 2.0, Variant.PR: 2.0, Variant.GV: 1.0,
            Variant.PIPE_PR_M: 1.5, Variant.PIPE_PR: 1.5}
    for v, t in want.items():
        assert iteration_time(v, p) == t


def test_zero_communication_and_zero_costs():
    p = CostParams(c_gr=0.0, t_mv=2.0, c_mv=0.5, t_2mv=3.0)
    assert iteration_time(Variant.HS, p) == iteration_time(Variant.PR, p)
    assert iteration_time(Variant.GV, p) == 2.5 and iteration_time(Variant.PIPE_PR, p) == 3.5
    assert all(iteration_time(v, CostParams()) == 0.0 for v in ALL)


def test_random_draws_match_hand_coded():
    rng = random.Random(123)
    for _ in range(100):
        t_mv = rng.uniform(0, 10)
        p = CostParams(rng.uniform(0, 10), t_mv, rng.uniform(0, 10), t_mv * rng.uniform(1, 2))
        p.validate()
        for v in ALL:
            assert iteration_time(v, p) == expected(v, p.c_gr, p.t_mv, p.c_mv, p.t_2mv)


def test_validation_and_scenarios():
    with pytest.raises(ValueError):
        CostParams(c_gr=-1.0).validate()
    with pytest.raises(ValueError):
        CostParams(0.0, 1.0, 0.0, 0.5).validate()
    with pytest.raises(ValueError):
        CostParams(0.0, 1.0, 0.0, 2.5).validate()
    with pytest.raises(ValueError):
        predict_scaling(Variant.HS, ScalingScenario())
    with pytest.raises(ValueError):
        predict_scaling(Variant.HS, ScalingScenario([2, 1], [CostParams(), CostParams()]))
    with pytest.raises(ValueError):
        predict_scaling(Variant.HS, ScalingScenario([1], [CostParams()]), iterations=0)
    # strong scaling: t_mv shrinks with nodes, c_gr grows -> GV overtakes HS
    s = ScalingScenario([1, 2, 4, 8], [CostParams(0.1 * n, 8.0 / n, 0.0, 12.0 / n) for n in (1, 2, 4, 8)])
    pts = predict_scaling(Variant.GV, s, 10)
    assert [p.nodes for p in pts] == [1, 2, 4, 8]
    assert pts[0].seconds == 10 * 8.0
    assert crossover_nodes(Variant.GV, Variant.HS, s) == 1
    assert crossover_nodes(Variant.HS, Variant.GV, s) is None


@pytest.mark.gpu
def test_device_calibration():
    P = pb.make_problem("p3", pb.poisson3d(48))
    A = cgvk.DeviceMatrix.from_csr(P.A)
    p, ms = calibrate(A, reps=20)
    assert ms["spmv"] > 0 and ms["block_spmv"] >= 0.5 * ms["spmv"] and ms["dot"] > 0 and ms["copy"] > 0
    assert p.t_mv <= p.t_2mv <= 2 * p.t_mv
    assert iteration_time(Variant.HS, p) > iteration_time(Variant.PR, p) >= iteration_time(Variant.GV, p)
