"""Device parity: the sm_100a engine, called through the package API (and so
through the C ABI), against the reference's own outputs (golden fixtures) and
against the CPU oracle.  Results must be bit-exact (integer/Boolean path)."""

import math
import threading

import numpy as np
import pytest

from fixtures import automaton, expected_reach, host_graph, oracle_graph, unpack_bits
from conftest import load_golden

import paper_2412_10287_b200 as P
from paper_2412_10287_b200 import datagen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def instances(reference_instances):
    return [(rec, host_graph(rec["graph"]), automaton(rec["nfa"])) for rec in reference_instances]


@pytest.mark.parametrize("algorithm,direction,kernel", [
    ("hybrid", "auto", "auto"), ("masked", "auto", "auto"), ("no_mask", "auto", "auto"),
    ("hybrid", "push", "auto"), ("hybrid", "pull", "auto"), ("masked", "pull", "auto"),
    ("hybrid", "auto", "grid"), ("masked", "push", "grid"), ("no_mask", "auto", "grid")])
def test_reference_instances(instances, algorithm, direction, kernel):
    """kernel="auto" runs these small instances on the single-CTA kernel
    (except forced pull); "grid" forces the persistent grid kernel."""
    opts = P.EngineOptions(algorithm=algorithm, timeout=math.inf, direction=direction, kernel=kernel)
    for rec, g, n in instances:
        res = P.eval_ssr(g, n, rec["source"], opts)
        assert np.array_equal(res.reach, expected_reach(rec, g.num_vertices)), rec["tag"]
        assert res.reachable == set(rec["expected"]), rec["tag"]
        assert res.iterations == rec["iterations"][algorithm], (rec["tag"], res.iterations)
        assert res.algorithm == algorithm


def test_sdr_duality(instances):
    opts = P.EngineOptions()
    for rec, g, n in instances:
        if "sdr_expected" not in rec:
            continue
        res = P.eval_sdr(g, n, rec["source"], opts)
        assert sorted(res.reachable) == rec["sdr_expected"], rec["tag"]
        assert res.iterations == rec["sdr_iterations"], rec["tag"]
        forced = P.eval_sdr(g, n, rec["source"], opts, "masked")
        assert forced.algorithm == "masked" and forced.reachable == res.reachable


def test_hybrid_thresholds(instances):
    for rec, g, n in instances:
        if "threshold_iterations" not in rec:
            continue
        for t, its in rec["threshold_iterations"].items():
            res = P.eval_ssr_hybrid(g, n, rec["source"], P.EngineOptions(switch_threshold=float(t)))
            assert res.reachable == set(rec["expected"]) and res.iterations == its


@pytest.mark.parametrize("kernel", ["auto", "grid"])
def test_debug_invariants(instances, kernel):
    opts = P.EngineOptions(debug_checks=True, kernel=kernel)
    for rec, g, n in instances[:200]:
        res = P.eval_ssr(g, n, rec["source"], opts)
        assert res.iterations <= n.nstates * g.num_vertices
        assert res.stats["visited_pairs"] == sum(res.stats["level_new"][: res.iterations + 1])


@pytest.mark.parametrize("kernel", ["auto", "grid"])
def test_timeout_raises(kernel):
    # test_engine.py:376-383
    nv = 3001
    g = P.LabeledGraph.from_edges(nv, ["a"], [(i, 0, i + 1) for i in range(3000)])
    n = P.Automaton.build(1, {(0, False): [(0, 0)]}, [0], [0])
    with pytest.raises(P.QueryTimeout) as ei:
        P.eval_ssr_masked(g, n, 0, P.EngineOptions(timeout=0.0, kernel=kernel))
    assert ei.value.iterations == 0
    res = P.eval_ssr_masked(g, n, 0, P.EngineOptions(timeout=math.inf, kernel=kernel))
    assert res.reachable == set(range(nv)) and res.iterations == nv
    # a deadline that expires mid-query is caught at an iteration boundary
    with pytest.raises(P.QueryTimeout) as ei:
        P.eval_ssr_masked(g, n, 0, P.EngineOptions(timeout=1e-4, kernel=kernel))
    assert 0 <= ei.value.iterations < nv


def test_empty_and_edge_cases():
    # no labels at all, single vertex (test_engine.py:127-134)
    g = P.LabeledGraph(1, [], [])
    n = P.Automaton.build(1, {(0, False): [(0, 0)]}, [0], [0])
    for alg in ("masked", "no_mask", "hybrid"):
        assert P.eval_ssr(g, n, 0, P.EngineOptions(algorithm=alg)).reachable == {0}
    # an automaton with no start state answers nothing; masked does 0 iterations,
    # the mask-free loops one (engine.py:157 vs :184, :209)
    g = P.LabeledGraph.from_edges(4, ["a"], [(0, 0, 1), (1, 0, 2)])
    n = P.Automaton.build(2, {(0, False): [(0, 1)]}, [], [1])
    assert P.eval_ssr_masked(g, n, 0, P.EngineOptions()).iterations == 0
    assert P.eval_ssr_hybrid(g, n, 0, P.EngineOptions()).iterations == 1
    assert P.eval_ssr_no_mask(g, n, 0, P.EngineOptions()).reachable == set()
    # multi-start, nondeterministic automaton
    n = P.Automaton.build(3, {(0, False): [(0, 1), (0, 2), (2, 2)], (0, True): [(1, 0)]},
                          [0, 2], [1, 2])
    og = oracle_graph({"nv": 4, "edges": [[(0, 1), (1, 2)]]})
    from oracle import OracleQuery, oracle_bfs

    oq = OracleQuery(n.to_json(), 1)
    for s in range(4):
        want, st = oracle_bfs(og, oq, s)
        got = P.eval_ssr(g, n, s, P.EngineOptions())
        assert np.array_equal(got.reach, want) and got.iterations == st["iterations"]


def test_concurrent_queries_deterministic(instances):
    rec, g, n = max(instances, key=lambda x: len(x[0]["expected"]))
    want = expected_reach(rec, g.num_vertices)
    errors = []

    def worker():
        try:
            for _ in range(20):
                r = P.eval_ssr(g, n, rec["source"], P.EngineOptions())
                assert np.array_equal(r.reach, want)
        except Exception as e:  # pragma: no cover - reported below
            errors.append(e)

    ts = [threading.Thread(target=worker) for _ in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors


def _config_case(name):
    gold = load_golden(f"{name}.json.gz")
    sg = datagen.generate(name)
    assert sg.digest() == gold["digest"], "generator drifted from the golden inputs"
    return gold, sg


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg5"])
def test_config_goldens(name):
    gold, sg = _config_case(name)
    g = sg.labeled_graph()
    for rec in gold["records"]:
        n = automaton(rec["nfa"])
        want = unpack_bits(rec["reach_bits"], sg.nv)
        assert int(want.sum()) == rec["reach_count"]
        for direction in ("auto", "push", "pull"):
            res = P.eval_ssr(g, n, rec["source"],
                             P.EngineOptions(timeout=math.inf, direction=direction))
            assert np.array_equal(res.reach, want), direction
            assert res.iterations == rec["iterations"]["hybrid"], direction


@pytest.mark.parametrize("direction", ["auto", "push", "pull", "grid-auto"])
@pytest.mark.parametrize("scale,seed,query", [
    (14, 21, "^a (b|c)* d"), (15, 22, "a ^b* c"), (16, 23, "a b*"),
    (13, 24, "(a|^b)* c+"), (12, 25, "(a ^a)* (b | c ^d)*"), (14, 26, "(a|b|c|d)*"),
    (13, 27, "a ^b c*")])
def test_rmat_vs_oracle(scale, seed, query, direction):
    import json
    import os

    from oracle import OracleGraph, OracleQuery, oracle_bfs

    sg = datagen.gen_rmat(scale, 16, 8, 1.0, seed)
    g = sg.labeled_graph()
    og = OracleGraph(sg.nv, sg.nl, sg.src, sg.dst, sg.lab)
    path = os.path.join(os.path.dirname(__file__), "golden", "extra_automata.json")
    nj = json.load(open(path))[query]
    n = automaton(nj)
    oq = OracleQuery(nj, sg.nl)
    deg = sg.out_degree()
    sources = [int(np.argmax(deg)), 0, sg.nv - 1, int(np.flatnonzero(deg)[len(np.flatnonzero(deg)) // 2])]
    for s in sources:
        want, st = oracle_bfs(og, oq, s)
        d, kernel = ("auto", "grid") if direction == "grid-auto" else (direction, "auto")
        got = P.eval_ssr(g, n, s, P.EngineOptions(timeout=math.inf, debug_checks=True,
                                                  direction=d, kernel=kernel))
        assert np.array_equal(got.reach, want), (query, s)
        assert got.iterations == st["iterations"]
        assert got.stats["te"] == st["te"]
        assert got.stats["visited_pairs"] == st["pairs"]
        # per-level push-model edges (pull levels too, under count_te) add up to TE (DFAs)
        dfa = all(np.all(np.diff(np.asarray(m.indptr)) <= 1) for m in n.transitions.values())
        if got.iterations < 64 and dfa:
            assert sum(got.stats["level_edges"][: got.iterations]) == st["te"], (query, s, direction)


def test_cfg3_golden():
    """R-MAT scale 24 (263M edges) against the reference's own answer."""
    gold, sg = _config_case("cfg3")
    g = sg.labeled_graph()
    for rec in gold["records"]:
        n = automaton(rec["nfa"])
        want = unpack_bits(rec["reach_bits"], sg.nv)
        for direction in ("auto", "push", "pull"):
            res = P.eval_ssr(g, n, rec["source"], P.EngineOptions(timeout=math.inf, direction=direction))
            assert np.array_equal(res.reach, want), direction
            assert res.iterations == rec["iterations"]["hybrid"], direction


def test_step_update_goldens():
    """step_update (engine.py:127-138) against the reference's own results."""
    from paper_2412_10287_b200.graph import CsrMatrix

    for rec in load_golden("step_update.json.gz"):
        g = host_graph(rec["graph"])
        n = automaton(rec["nfa"])
        shape = (n.nstates, g.num_vertices)
        m = CsrMatrix.from_pairs(*shape, [tuple(x) for x in rec["m"]])
        p = CsrMatrix.from_pairs(*shape, [tuple(x) for x in rec["p"]])
        out = P.step_update(m, p, g, n, P.EngineOptions())
        assert isinstance(out, CsrMatrix)
        assert out.pairs() == [tuple(x) for x in rec["expected"]], rec["tag"]


@pytest.mark.parametrize("seed", [41, 42])
def test_device_ingest_matches_host_csr(seed):
    """rpq_graph_create_coo: per-label CSR built on the device (dedup, rows
    sorted, self-loops kept) equals the oracle's independent host build, and
    queries over it give the same answers as over the uploaded host CSR."""
    from oracle import OracleGraph, OracleQuery, oracle_bfs

    rng = np.random.default_rng(seed)
    nv, nl, ne = 3000, 5, 40000
    src = rng.integers(0, nv, ne).astype(np.int32)
    dst = rng.integers(0, nv, ne).astype(np.int32)
    lab = (rng.zipf(1.5, ne) % nl).astype(np.int32)
    src[:500] = dst[:500]          # self-loops
    src[500:1500] = src[1500:2500]  # duplicates
    dst[500:1500] = dst[1500:2500]
    lab[500:1500] = lab[1500:2500]
    g = P.LabeledGraph.from_coo(nv, list("abcde"), src, dst, lab)
    dg = P.DeviceGraph(g, ingest="coo")
    og = OracleGraph(nv, nl, src, dst, lab)
    dg.ensure_labels(range(nl))
    for l in range(nl):
        for inv in (False, True):
            rowptr, col = dg.label_csr(l, inv)
            indptr, indices = og.slot_csr(l, inv)
            assert np.array_equal(rowptr.astype(np.int64), indptr), (l, inv)
            assert np.array_equal(col, indices), (l, inv)
    import json
    import os

    autos = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "extra_automata.json")))
    for query in ("a ^b* c", "(a|^b)* c+", "(a b)* | (c ^d)+ e?"):
        n = automaton(autos[query])
        oq = OracleQuery(autos[query], nl)
        for s in (0, 17, nv - 1):
            want, st = oracle_bfs(og, oq, s)
            got = P.eval_ssr(dg, n, s, P.EngineOptions(timeout=math.inf))
            assert np.array_equal(got.reach, want) and got.iterations == st["iterations"]


def test_queries_with_different_shared_memory_interleave():
    """The kernels' dynamic shared memory limit is per function: a query
    created after another with a smaller table must not shrink the limit the
    first one launches with (run big, small, big on the grid kernel)."""
    import json
    import os

    from oracle import OracleGraph, OracleQuery, oracle_bfs

    sg = datagen.gen_rmat(13, 16, 8, 1.0, 31)
    g = sg.labeled_graph()
    og = OracleGraph(sg.nv, sg.nl, sg.src, sg.dst, sg.lab)
    path = os.path.join(os.path.dirname(__file__), "golden", "extra_automata.json")
    table = json.load(open(path))
    opts = P.EngineOptions(timeout=math.inf, kernel="grid")
    want, nfa = {}, {}
    for query in ("(a ^a)* (b | c ^d)*", "a b*", "(a ^a)* (b | c ^d)*", "a b*"):
        nj = table[query]
        if query not in want:  # same automaton objects: the cached queries are reused
            want[query] = oracle_bfs(og, OracleQuery(nj, sg.nl), 0)[0]
            nfa[query] = automaton(nj)
        got = P.eval_ssr(g, nfa[query], 0, opts)
        assert np.array_equal(got.reach, want[query]), query


def test_zero_copy_statistics_match_the_copy_path():
    """RPQ_TUNE_ZERO_COPY: the grid kernel's last CTA writes the statistics
    block into pinned host memory instead of a copy node; both paths report
    the same run (answer, levels, counts), run after run."""
    from paper_2412_10287_b200 import _lib

    sg = datagen.gen_rmat(14, 16, 8, 1.0, 41)
    g = sg.labeled_graph()
    import json
    import os

    path = os.path.join(os.path.dirname(__file__), "golden", "extra_automata.json")
    n = automaton(json.load(open(path))["^a (b|c)* d"])
    src = int(np.argmax(sg.out_degree()))
    pq = P.PreparedQuery(g, n)
    pq.set_tuning(kernel="grid")
    seen = []
    for zc in (0, 1, 0, 1, 1):
        assert _lib.engine().rpq_query_set_tuning(pq.q, _lib.TUNE_ZERO_COPY, float(zc)) == 0, _lib.last_error()
        pq.launch(src)
        st = pq.wait().to_dict()
        keep = {k: st[k] for k in ("status", "iterations", "levels", "te", "visited_pairs", "reach_count",
                                   "level_new", "level_dir")}
        seen.append((keep, pq.reach().copy()))
    for keep, reach in seen[1:]:
        assert keep == seen[0][0]
        assert np.array_equal(reach, seen[0][1])
    assert seen[0][0]["reach_count"] == int(seen[0][1].sum()) > 0
    pq.close()
