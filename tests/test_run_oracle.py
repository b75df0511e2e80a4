"""Pins oracle/run.py (the restated run() driver + probes) against the
reference's own run(): tests/golden/run_records.json was produced by
proj/src/runner.cpp through oracle/_ref (scripts/make_golden.py run). With
the sequential dot the restatement must reproduce every record field, the
final status and the summary bit for bit."""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from oracle import run as ORUN
from paper_1905_01549_b200 import problems as pb

from conftest import GOLDEN

with open(os.path.join(GOLDEN, "run_records.json")) as f:
    GOLD = json.load(f)

PROBLEMS = {"p2d_24": pb.make_problem("p2d_24", pb.poisson2d(24)),
            "rs_600": pb.make_problem("rs_600", pb.random_spd(600, 7, 90, 5))}


def stop_of(case):
    s = case["stop"]
    return (s[0], s[1]) if len(s) == 2 else (s[0], s[1], s[2])


def unhex(v):
    return None if v is None else float.fromhex(v)


@pytest.mark.parametrize("key", sorted(GOLD["cases"]))
def test_restated_run_matches_reference(key):
    case = GOLD["cases"][key]
    P = PROBLEMS[case["problem"]]
    got = ORUN.run(P.A, case["variant"], case["precond"], P.b, P.x0, case["max_iter"], stop_of(case),
                   case["probes"], case["cadence"], P.x_star, mode="seq")
    assert (got["state"], got["breakdown"], got["criterion"]) == \
        (case["state"], case["breakdown"], case["criterion"])
    assert len(got["records"]) == len(case["records"])
    for rec, gold in zip(got["records"], case["records"]):
        assert rec["k"] == gold[0]
        for f, gv in zip(GOLD["fields"], gold[1:]):
            want = unhex(gv)
            have = rec[f]
            assert (have is None) == (want is None), (key, rec["k"], f)
            if want is not None:
                assert np.float64(have).view(np.int64) == np.float64(want).view(np.int64), \
                    (key, rec["k"], f, have, want)
    if case["summary"] is None:
        assert got["summary"] is None
    else:
        assert got["summary"]["iters_to_1e5"] == case["summary"]["iters_to_1e5"]
        assert got["summary"]["min_log10_err"] == case["summary"]["min_log10_err"]


def test_restated_run_errors():
    P = PROBLEMS["p2d_24"]
    with pytest.raises(ValueError):
        ORUN.run(P.A, 0, 0, P.b, P.x0, -1, ("fixed", 5))
    with pytest.raises(ValueError):
        ORUN.run(P.A, 0, 0, P.b, P.x0, 5, ("error", 1e-5))
    with pytest.raises(ValueError):
        ORUN.run(P.A, 0, 0, P.b, P.x0, 5, ("fixed", 5), x_star=P.x0)
