"""The bench front end on the device (paper_2412_10287_b200/cli.py), with the
reference's CLI cases (test_cli.py:101-158) and the desk-scale workload
(test_acceptance.py:238-335) whose rows must carry the reference's own
result counts and iteration counts."""

import csv
import io
import math

import pytest

from fixtures import automaton, desk_bench, desk_host_graph

import paper_2412_10287_b200 as P
from paper_2412_10287_b200 import cli

pytestmark = pytest.mark.gpu

# test_cli.py:17 TRIANGLE: 3 -a-> 4, 4 -a-> 3, 3 -b-> 5 (vertices named in order of appearance)
TRI_VERTICES = ["3", "4", "5"]


def triangle():
    from paper_2412_10287_b200.graph import CsrMatrix

    a = CsrMatrix.from_pairs(3, 3, [(0, 1), (1, 0)])
    b = CsrMatrix.from_pairs(3, 3, [(0, 2)])
    return P.LabeledGraph(3, ["a", "b"], [a, b], vertices=TRI_VERTICES)


def tri_compiler():
    # the reference compiler's automata (extra_automata.json: labels a=0, b=1, ...)
    import json
    import os

    here = os.path.dirname(os.path.abspath(__file__))
    extra = json.load(open(os.path.join(here, "golden", "extra_automata.json")))
    table = {p: automaton(nj) for p, nj in extra.items()}
    return lambda pattern: table[pattern]


def test_bench_rows_and_errors():
    g = triangle()
    comp = tri_compiler()
    entries = cli.parse_workload(io.StringIO(
        "q1\tssr\t3\ta b*\nbad-vertex\tssr\t42\ta\nbad-pattern\tssr\t3\ta )b\nq3\tssr\t4\ta+ b\n"))
    rows = cli.run_bench(g, entries, P.EngineOptions(), compile_fn=comp)
    assert [r["status"] for r in rows] == ["ok", "error", "error", "ok"]
    assert rows[0]["result_count"] == 1  # a b* from 3 reaches exactly vertex 4
    assert rows[3]["result_count"] == 1  # a+ b from 4: {5}
    out = io.StringIO()
    cli.write_csv(rows, out)
    got = list(csv.reader(io.StringIO(out.getvalue())))
    assert got[0] == cli.BENCH_HEADER and len(got) == 5


def test_bench_repeat_parallel_and_extended():
    g = triangle()
    comp = tri_compiler()
    entries = cli.parse_workload(io.StringIO("".join(f"q{i}\tssr\t3\ta+ b\n" for i in range(4))))
    rows = cli.run_bench(g, entries, P.EngineOptions(), repeat=3, workers=2, compile_fn=comp, work=True)
    assert [r["id"] for r in rows] == ["q0", "q1", "q2", "q3"]
    assert all(r["result_count"] == 1 and r["status"] == "ok" for r in rows)
    assert all(r["te"] >= 1 and r["levels"] == r["iterations"] and r["bytes_alg"] > 0 for r in rows)


def test_bench_timeout_status():
    from paper_2412_10287_b200.graph import CsrMatrix

    nv = 3001
    chain = CsrMatrix.from_pairs(nv, nv, [(i, i + 1) for i in range(3000)])
    g = P.LabeledGraph(nv, ["a"], [chain])
    a_star = P.Automaton.build(1, {(0, False): [(0, 0)]}, [0], [0])
    entries = cli.parse_workload(io.StringIO("slow\tssr\t0\ta*\n"))
    rows = cli.run_bench(g, entries, P.EngineOptions(timeout=0.001, kernel="grid"),
                         compile_fn=lambda _p: a_star)
    assert rows[0]["status"] == "timeout" and rows[0]["time_ms"] == 1.0


def test_desk_workload_rows_match_reference():
    """All 1,000 desk entries through run_bench (hybrid): result counts and
    iteration counts equal the reference's."""
    rec, csr = desk_bench()
    g = desk_host_graph(rec, csr)
    autos = {pat: automaton(nj) for pat, nj in rec["automata"].items()}
    entries = [cli.WorkloadEntry(e["id"], e["mode"], str(e["vertex"]), e["pattern"]) for e in rec["entries"]]
    rows = cli.run_bench(g, entries, P.EngineOptions(timeout=math.inf), compile_fn=autos.__getitem__)
    for e, r in zip(rec["entries"], rows):
        assert r["status"] == "ok" and r["id"] == e["id"]
        assert r["result_count"] == e["count"], e["id"]
        assert r["iterations"] == e["iterations"]["hybrid"], e["id"]


def test_batch_rows_match_single_source():
    rec, csr = desk_bench()
    g = desk_host_graph(rec, csr)
    pat = rec["entries"][0]["pattern"]
    n = automaton(rec["automata"][pat])
    ents = [e for e in rec["entries"] if e["pattern"] == pat and e["mode"] == "ssr"]
    rows = cli.run_batch(g, n, [e["vertex"] for e in ents], P.EngineOptions(timeout=math.inf), repeat=2)
    for e, r in zip(ents, rows):
        assert r["result_count"] == e["count"] and r["iterations"] == e["iterations"]["masked"], e["id"]
        assert r["te"] >= 0 and r["gteps"] >= 0
