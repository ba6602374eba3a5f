"""Multi-source batches (eval_ssr_batch): row s of the batch
answer must equal the single-source answer from sources[s] -- checked against
the reference's own outputs (golden fixtures) and the CPU oracle, bit-exact.
The batch kernel shares frontier rows between sources (bit-sliced words), so
these tests mix sources whose frontiers overlap, duplicates, and sources with
no start transition."""

import json
import math
import os

import numpy as np
import pytest

from fixtures import automaton, expected_reach, host_graph
from conftest import load_golden

import paper_2412_10287_b200 as P
from paper_2412_10287_b200 import datagen

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _autos():
    return json.load(open(os.path.join(GOLDEN, "extra_automata.json")))


def test_reference_instances_batched(reference_instances):
    """Group the reference's instances by (graph, automaton): every instance's
    source goes into one batch per group, padded with every other vertex."""
    opts = P.EngineOptions(timeout=math.inf)
    for rec in reference_instances[:400]:
        g, n = host_graph(rec["graph"]), automaton(rec["nfa"])
        nv = g.num_vertices
        srcs = [rec["source"]] + [v for v in range(min(nv, 40)) if v != rec["source"]]
        stats = []
        got = P.eval_ssr_batch(g, n, srcs, opts, stats=stats)
        assert got.shape == (len(srcs), nv)
        assert np.array_equal(got[0], expected_reach(rec, nv)), rec["tag"]
        # the other rows against the single-source engine (itself pinned above)
        for i, s in enumerate(srcs[1:], 1):
            assert np.array_equal(got[i], P.eval_ssr(g, n, s, opts).reach), (rec["tag"], s)
        # masked-loop iteration count of the first source
        its = stats[0]["iterations"][0]
        assert its == rec["iterations"]["masked"], (rec["tag"], its)


@pytest.mark.parametrize("scale,seed,query", [
    (14, 21, "^a (b|c)* d"), (15, 22, "a ^b* c"), (13, 24, "(a|^b)* c+"),
    (12, 25, "(a ^a)* (b | c ^d)*"), (14, 26, "(a|b|c|d)*"), (13, 27, "a ^b c*")])
def test_rmat_batch_vs_oracle(scale, seed, query):
    from oracle import OracleGraph, OracleQuery, oracle_bfs

    sg = datagen.gen_rmat(scale, 16, 8, 1.0, seed)
    g = sg.labeled_graph()
    og = OracleGraph(sg.nv, sg.nl, sg.src, sg.dst, sg.lab)
    nj = _autos()[query]
    n = automaton(nj)
    oq = OracleQuery(nj, sg.nl)
    deg = sg.out_degree()
    rng = np.random.default_rng(seed)
    nz = np.flatnonzero(deg)
    # BATCH + 5 sources: two launches (the second partial); hubs, a
    # duplicate, isolated vertices, randoms
    srcs = [int(np.argmax(deg)), 0, 0, sg.nv - 1] + [int(x) for x in rng.choice(nz, P._lib.BATCH + 1)]
    stats = []
    got = P.eval_ssr_batch(g, n, srcs, P.EngineOptions(timeout=math.inf), stats=stats)
    assert len(stats) == 2
    te = pairs = 0
    for i, s in enumerate(srcs):
        want, st = oracle_bfs(og, oq, s)
        assert np.array_equal(got[i], want), (query, i, s)
        b, k = divmod(i, P._lib.BATCH)
        assert stats[b]["iterations"][k] == st["iterations"], (query, s)
        assert stats[b]["reach_count"][k] == int(want.sum())
        te += st["te"]
        pairs += st["pairs"]
    assert sum(x["te"] for x in stats) == te
    assert sum(x["visited_pairs"] for x in stats) == pairs


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg5"])
def test_config_goldens_batched(name):
    gold = load_golden(f"{name}.json.gz")
    sg = datagen.generate(name)
    assert sg.digest() == gold["digest"]
    g = sg.labeled_graph()
    from fixtures import unpack_bits

    by_query = {}
    for rec in gold["records"]:
        by_query.setdefault(json.dumps(rec["nfa"], sort_keys=True), []).append(rec)
    for recs in by_query.values():
        n = automaton(recs[0]["nfa"])
        srcs = [r["source"] for r in recs]
        got = P.eval_ssr_batch(g, n, srcs, P.EngineOptions(timeout=math.inf))
        for i, r in enumerate(recs):
            assert np.array_equal(got[i], unpack_bits(r["reach_bits"], sg.nv)), (name, r["source"])


def test_batch_edge_cases():
    n = P.Automaton.build(1, {(0, False): [(0, 0)]}, [0], [0])
    g = P.LabeledGraph.from_edges(5, ["a"], [(0, 0, 1), (1, 0, 2), (3, 0, 3)])
    assert P.eval_ssr_batch(g, n, [], P.EngineOptions()).shape == (0, 5)
    got = P.eval_ssr_batch(g, n, [0, 2, 3, 4, 0], P.EngineOptions())
    assert got.tolist() == [[1, 1, 1, 0, 0], [0, 0, 1, 0, 0], [0, 0, 0, 1, 0],
                            [0, 0, 0, 0, 1], [1, 1, 1, 0, 0]]
    with pytest.raises(IndexError):
        P.eval_ssr_batch(g, n, [0, 5], P.EngineOptions())
    with pytest.raises(IndexError):
        P.eval_ssr_batch(g, n, [-1], P.EngineOptions())
    with pytest.raises(P.QueryTimeout):
        P.eval_ssr_batch(g, n, [0], P.EngineOptions(timeout=0.0))
    # no start state: every answer is empty
    n0 = P.Automaton.build(1, {(0, False): [(0, 0)]}, [], [0])
    assert P.eval_ssr_batch(g, n0, [0, 1], P.EngineOptions()).sum() == 0
    # a label the graph does not have (engine.py:100-101) and a final-only start
    n2 = P.Automaton.build(2, {(0, False): [(0, 1)], (7, False): [(1, 1)]}, [0], [0, 1])
    got = P.eval_ssr_batch(g, n2, [0, 1, 3], P.EngineOptions())
    for i, s in enumerate([0, 1, 3]):
        assert np.array_equal(got[i], P.eval_ssr(g, n2, s, P.EngineOptions()).reach)


def test_batch_long_chain_and_timeout():
    nv = 3001
    g = P.LabeledGraph.from_edges(nv, ["a"], [(i, 0, i + 1) for i in range(3000)])
    n = P.Automaton.build(1, {(0, False): [(0, 0)]}, [0], [0])
    stats = []
    got = P.eval_ssr_batch(g, n, [0, 1500, 3000], P.EngineOptions(timeout=math.inf), stats=stats)
    assert got.sum(axis=1).tolist() == [3001, 1501, 1]
    assert stats[0]["iterations"] == [3001, 1501, 1]
    with pytest.raises(P.QueryTimeout):
        P.eval_ssr_batch(g, n, [0], P.EngineOptions(timeout=1e-4))
    # the query object is still usable after a timeout
    assert P.eval_ssr_batch(g, n, [2990], P.EngineOptions(timeout=math.inf)).sum() == 11


def test_batch_hub_rows_split():
    """A star with a 100k-edge hub row (heavy chunks) and a 2-hop fan-out."""
    nv = 200_001
    hub = [(0, 0, v) for v in range(1, 100_001)]
    fan = [(v, 1, 100_000 + v) for v in range(1, 100_001)]
    g = P.LabeledGraph.from_edges(nv, ["a", "b"], hub + fan)
    n = automaton(_autos()["a b*"]) if "a b*" in _autos() else None
    if n is None:
        n = P.Automaton.build(2, {(0, False): [(0, 1)], (1, False): [(1, 1)]}, [0], [1])
    srcs = [0, 0, 5, 100_005]
    got = P.eval_ssr_batch(g, n, srcs, P.EngineOptions(timeout=math.inf))
    for i, s in enumerate(srcs):
        assert np.array_equal(got[i], P.eval_ssr(g, n, s, P.EngineOptions(timeout=math.inf)).reach)
