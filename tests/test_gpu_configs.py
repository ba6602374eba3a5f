"""Full-size parity on the BASELINE configs the per-query suites do not cover
in full (north_star: "bit-exact reachable sets on all five configs"):

* cfg5 -- the 16-32-state wording of BASELINE.json: the reference compiler's
  unminimized automata (17 states for the forward and the ^a_even chains, 25
  for the (a_even|^a_even)* variant, query_compiler.py:477-485 minimize=False)
  against the reference's own answers (tests/golden/cfg5_raw.json.gz), single
  source and batched; and all 1,024 bench sources of the 9-state chain
  through the batch kernel against the CPU oracle (threaded), plus 256 / 64
  sources of the raw two-way automata.
* cfg4 -- Chung-Lu 90M vertices / 1.05B deduplicated edges, 2,000 labels:
  the 4 templates x 32 uniform sources against the CPU oracle over the 4
  query labels (result-identical: _label_pairs touches only alphabet labels,
  engine.py:99-102), and against the reference's own answers where
  tests/golden/cfg4.json.gz holds them.

The oracle (oracle/rpq_oracle.c oracle_bfs) is pinned to the reference by
tests/test_oracle_golden.py.  These runs take minutes: marked slow."""

import json
import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from conftest import GOLDEN, load_golden
from fixtures import automaton, reach_sha256, unpack_bits

import paper_2412_10287_b200 as P
from paper_2412_10287_b200 import datagen

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
AUTOS = os.path.join(ROOT, "paper_2412_10287_b200", "data", "config_automata.json")
THREADS = max(1, min(32, os.cpu_count() or 1))


def _oracle_all(og, nj, nl, sources):
    """oracle_bfs over `sources` on all host threads -> {source: (reach, stats)}."""
    from oracle import OracleQuery, oracle_bfs

    oq = OracleQuery(nj, nl)
    oq.prepare(og)
    uniq = sorted(set(sources))
    with ThreadPoolExecutor(max_workers=THREADS) as pool:
        res = list(pool.map(lambda s: oracle_bfs(og, oq, s), uniq))
    return dict(zip(uniq, res))


@pytest.fixture(scope="module")
def cfg5():
    sg = datagen.generate("cfg5")
    return sg, sg.labeled_graph()


def test_cfg5_raw_automata_goldens(cfg5):
    """17- and 25-state automata (unminimized) vs the reference's answers."""
    sg, g = cfg5
    gold = load_golden("cfg5_raw.json.gz")
    assert sg.digest() == gold["digest"]
    nstates = set()
    by_query = {}
    for rec in gold["records"]:
        n = automaton(rec["nfa"])
        nstates.add(n.nstates)
        want = unpack_bits(rec["reach_bits"], sg.nv)
        assert int(want.sum()) == rec["reach_count"]
        for direction in ("auto", "push", "pull"):
            res = P.eval_ssr(g, n, rec["source"], P.EngineOptions(timeout=math.inf, direction=direction))
            assert np.array_equal(res.reach, want), (rec["query"], rec["source"], direction)
            assert res.iterations == rec["iterations"]["hybrid"], (rec["query"], direction)
        by_query.setdefault(rec["query"], []).append(rec)
    assert nstates == {17, 25}
    for recs in by_query.values():
        n = automaton(recs[0]["nfa"])
        rows = P.eval_ssr_batch(g, n, [r["source"] for r in recs], P.EngineOptions(timeout=math.inf))
        for row, r in zip(rows, recs):
            assert np.array_equal(row, unpack_bits(r["reach_bits"], sg.nv)), ("batch", r["query"])


@pytest.mark.parametrize("query,kind,count", [
    (datagen.CHAIN16, "min", 1024),
    (datagen.CHAIN16_TWOWAY, "raw", 256),
    (datagen.CHAIN16_BOTHWAY, "raw", 64),
])
def test_cfg5_bench_sources_batched(cfg5, query, kind, count):
    """BASELINE cfg5: the first `count` of the 1,024 uniform sources through
    eval_ssr_batch (64 per launch) vs the oracle: answers, per-source
    iteration counts, and the batch's summed TE and |P|."""
    from oracle import OracleGraph

    sg, g = cfg5
    nj = json.load(open(AUTOS))["cfg5"][f"{query}|{kind}"]
    n = automaton(nj)
    srcs = datagen.pick_sources(sg, "cfg5", count=count)
    og = OracleGraph(sg.nv, sg.nl, sg.src, sg.dst, sg.lab)
    want = _oracle_all(og, nj, sg.nl, srcs)
    stats = []
    rows = P.eval_ssr_batch(g, n, srcs, P.EngineOptions(timeout=math.inf), stats=stats)
    te = pairs = 0
    for i, s in enumerate(srcs):
        w, st = want[s]
        assert np.array_equal(rows[i], w), (query, kind, s)
        b = stats[i // P._lib.BATCH]
        assert b["iterations"][i % P._lib.BATCH] == st["iterations"], (query, s)
        te += st["te"]
        pairs += st["pairs"]
    assert sum(x["te"] for x in stats) == te
    assert sum(x["visited_pairs"] for x in stats) == pairs


@pytest.fixture(scope="module")
def cfg4():
    from oracle import OracleGraph

    sg = datagen.generate("cfg4")
    g = sg.labeled_graph()  # device ingest from the edge list (all 2,000 labels)
    keep = sg.lab < 4
    og = OracleGraph(sg.nv, 4, sg.src[keep], sg.dst[keep], sg.lab[keep])
    srcs = datagen.pick_sources(sg, "cfg4", count=32)
    return sg, g, og, srcs


@pytest.mark.parametrize("query", datagen.CONFIGS["cfg4"]["queries"])
def test_cfg4_templates_vs_oracle(cfg4, query):
    """The 4 templates x 32 uniform non-isolated sources, single-source
    (grid kernel, auto direction) and batched, vs the oracle; sources the
    reference itself evaluated (cfg4.json.gz) also vs its answer digests."""
    sg, g, og, srcs = cfg4
    nj = json.load(open(AUTOS))["cfg4"][f"{query}|min"]
    n = automaton(nj)
    want = _oracle_all(og, nj, 4, srcs)
    opts = P.EngineOptions(timeout=math.inf)
    for s in srcs:
        w, st = want[s]
        res = P.eval_ssr(g, n, s, opts)
        assert np.array_equal(res.reach, w), (query, s)
        assert res.iterations == st["iterations"], (query, s)
    rows = P.eval_ssr_batch(g, n, srcs, opts)
    for row, s in zip(rows, srcs):
        assert np.array_equal(row, want[s][0]), ("batch", query, s)
    if os.path.exists(os.path.join(GOLDEN, "cfg4.json.gz")):
        gold = load_golden("cfg4.json.gz")
        assert gold["digest"] == sg.digest()
        checked = 0
        for rec in gold["records"]:
            if rec["query"] != query:
                continue
            res = P.eval_ssr(g, n, rec["source"], opts)
            assert int(res.reach.sum()) == rec["reach_count"], (query, rec["source"])
            assert reach_sha256(res.reach) == rec["reach_sha256"], (query, rec["source"])
            assert res.iterations == rec["iterations"]["hybrid"], (query, rec["source"])
            checked += 1
        assert checked >= 2
