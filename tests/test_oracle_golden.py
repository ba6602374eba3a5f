"""Pin the CPU oracle (oracle/rpq_oracle.c) to the reference's own outputs.

Every record in tests/golden/reference_instances.json.gz was produced by
running /root/reference/pkg/src/rpq (tests/golden/make_golden.py) on the
RNG streams of the reference's tests; both oracle entry points must reproduce
the reference's answer sets and iteration counts exactly.
"""

import math

import numpy as np
import pytest

from fixtures import expected_reach, oracle_graph
from oracle import OracleQuery, oracle_bfs, oracle_port


def _reverse_json(nj):
    """query_compiler.py:488-502 on the fixture format."""
    return {
        "nstates": nj["nstates"],
        "transitions": [[t[0], not t[1], [[b, a] for a, b in t[2]]] for t in nj["transitions"]],
        "alphabet": [[t[0], not t[1]] for t in nj["transitions"]],
        "starts": nj["finals"],
        "finals": nj["starts"],
    }


def test_fixture_counts(reference_instances):
    tags = [r["tag"].split("/")[0] for r in reference_instances]
    assert tags.count("engine_random_15") == 40
    assert tags.count("acceptance_c1") == 500
    assert tags.count("acceptance_c2") == 100
    assert tags.count("acceptance_c4") == 100
    assert tags.count("hybrid_9") == 15
    assert tags.count("known") >= 10


def test_bfs_matches_reference(reference_instances):
    for rec in reference_instances:
        g = oracle_graph(rec["graph"])
        q = OracleQuery(rec["nfa"], len(rec["graph"]["labels"]))
        reach, st = oracle_bfs(g, q, rec["source"])
        assert np.array_equal(reach, expected_reach(rec, g.nv)), rec["tag"]
        assert st["iterations"] == rec["iterations"]["masked"], rec["tag"]
        # the reference's own set-based oracle agrees (compiled automata)
        assert sorted(np.flatnonzero(reach).tolist()) == rec["oracle_ssr"], rec["tag"]


@pytest.mark.parametrize("algorithm", ["masked", "no_mask", "hybrid"])
def test_port_matches_reference(reference_instances, algorithm):
    for rec in reference_instances:
        g = oracle_graph(rec["graph"])
        q = OracleQuery(rec["nfa"], len(rec["graph"]["labels"]))
        reach, st = oracle_port(g, q, rec["source"], algorithm)
        assert np.array_equal(reach, expected_reach(rec, g.nv)), (rec["tag"], algorithm)
        assert st["iterations"] == rec["iterations"][algorithm], (rec["tag"], algorithm)


def test_port_hybrid_thresholds(reference_instances):
    for rec in reference_instances:
        if not rec["tag"].startswith("hybrid_9/"):
            continue
        g = oracle_graph(rec["graph"])
        q = OracleQuery(rec["nfa"], len(rec["graph"]["labels"]))
        for t, its in rec["threshold_iterations"].items():
            reach, st = oracle_port(g, q, rec["source"], "hybrid", threshold=float(t))
            assert np.array_equal(reach, expected_reach(rec, g.nv))
            assert st["iterations"] == its


def test_sdr_duality(reference_instances):
    for rec in reference_instances:
        if "sdr_expected" not in rec:
            continue
        g = oracle_graph(rec["graph"])
        q = OracleQuery(_reverse_json(rec["nfa"]), len(rec["graph"]["labels"]))
        reach, st = oracle_bfs(g, q, rec["source"])
        assert sorted(np.flatnonzero(reach).tolist()) == rec["sdr_expected"], rec["tag"]
        assert st["iterations"] == rec["sdr_iterations"], rec["tag"]


def test_known_answers(reference_instances):
    known = {r["tag"]: r for r in reference_instances if r["tag"].startswith("known/")}
    assert known["known/triangle a* b from 3"]["expected_names"] == ["5"]
    assert known["known/chain a+"]["expected_names"] == ["v1", "v2"]
    assert "3" in known["known/inverse a ^a"]["expected_names"]
    assert known["known/absent label"]["expected"] == []
    assert known["known/no a-edges a*"]["expected_names"] == ["0"]
    assert len(known["known/41-vertex chain a*"]["expected"]) == 41
    for rec in known.values():
        g = oracle_graph(rec["graph"])
        q = OracleQuery(rec["nfa"], len(rec["graph"]["labels"]))
        reach, _ = oracle_bfs(g, q, rec["source"])
        assert np.array_equal(reach, expected_reach(rec, g.nv)), rec["tag"]


def test_bad_source_raises(reference_instances):
    rec = reference_instances[0]
    g = oracle_graph(rec["graph"])
    q = OracleQuery(rec["nfa"], len(rec["graph"]["labels"]))
    with pytest.raises(IndexError):
        oracle_bfs(g, q, g.nv)
    with pytest.raises(IndexError):
        oracle_port(g, q, -1)


def test_port_timeout(reference_instances):
    # 3000-vertex chain under a*: the reference raises at timeout=0 (test_engine.py:376-383)
    from oracle import OracleGraph

    nv = 3001
    g = OracleGraph(nv, 1, np.arange(3000, dtype=np.int32), np.arange(1, 3001, dtype=np.int32),
                    np.zeros(3000, dtype=np.int32))
    q = OracleQuery({"nstates": 1, "transitions": [[0, False, [[0, 0]]]], "alphabet": [[0, False]],
                     "starts": [0], "finals": [0]}, 1)
    with pytest.raises(TimeoutError):
        oracle_port(g, q, 0, "masked", timeout=0.0)
    reach, st = oracle_port(g, q, 0, "masked", timeout=math.inf)
    assert reach.sum() == nv and st["iterations"] == nv + 0  # 3000 steps + final empty one


def test_desk_bench_oracle():
    """Criterion 7's 1,000-entry workload (test_acceptance.py:238-335): both
    oracle entry points reproduce the reference's answers (sha256 of the
    sorted ids) and every algorithm's iteration count."""
    from fixtures import answer_digest, desk_bench, desk_oracle_graph

    rec, csr = desk_bench()
    assert len(rec["entries"]) == 1000 and rec["num_edges"] > 900_000
    og = desk_oracle_graph(rec, csr)
    nl = len(rec["labels"])
    queries = {}
    for e in rec["entries"]:
        key = (e["pattern"], e["mode"])
        if key not in queries:
            nj = rec["automata"][e["pattern"]]
            queries[key] = OracleQuery(nj if e["mode"] == "ssr" else _reverse_json(nj), nl)
        oq = queries[key]
        reach, st = oracle_bfs(og, oq, e["vertex"])
        assert int(reach.sum()) == e["count"] and answer_digest(reach) == e["sha256"], e["id"]
        assert st["iterations"] == e["iterations"]["masked"], e["id"]
        for alg in ("no_mask", "hybrid"):
            r2, s2 = oracle_port(og, oq, e["vertex"], alg)
            assert np.array_equal(r2, reach) and s2["iterations"] == e["iterations"][alg], (e["id"], alg)
