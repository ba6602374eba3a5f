"""The plan evaluator (eval_plan, engine.py:292-390) on the device against the
reference's own outputs: answers and closure-round counts for source- and
destination-bound walks (tests/golden/plan.json.gz, made by running the
reference on the RNG streams of its own tests)."""

import math

import numpy as np
import pytest

from fixtures import host_graph
from conftest import load_golden

import paper_2412_10287_b200 as P
from paper_2412_10287_b200 import plan

pytestmark = pytest.mark.gpu


def test_plan_goldens():
    recs = load_golden("plan.json.gz")
    assert len(recs) >= 240
    opts = P.EngineOptions(timeout=math.inf)
    for rec in recs:
        g = host_graph(rec["graph"])
        ast = plan.ast_from_json(rec["ast"])
        for mode in ("source", "destination"):
            res = plan.eval_plan(g, ast, (mode, rec["vertex"]), opts)
            assert sorted(res.reachable) == rec[mode]["reach"], (rec["tag"], mode)
            assert res.iterations == rec[mode]["iterations"], (rec["tag"], mode)
            assert res.algorithm == "plan"


def test_plan_timeout_and_validation():
    nv = 3001
    g = P.LabeledGraph.from_edges(nv, ["a"], [(i, 0, i + 1) for i in range(3000)])
    ast = plan.Star(plan.Label("a"))
    with pytest.raises(P.QueryTimeout):  # test_engine.py:330
        plan.eval_plan(g, ast, ("source", 0), P.EngineOptions(timeout=0.0))
    res = plan.eval_plan(g, ast, ("source", 2990), P.EngineOptions(timeout=math.inf))
    assert res.reachable == set(range(2990, nv)) and res.iterations == 11
    with pytest.raises(ValueError):
        plan.eval_plan(g, ast, ("middle", 0), P.EngineOptions())
    with pytest.raises(IndexError):
        plan.eval_plan(g, ast, ("source", nv), P.EngineOptions())
