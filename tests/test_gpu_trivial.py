"""Sources none of whose seed rows has an edge are answered on the host by the
fused eval call (no launch): P is the seed, one iteration (none without a start
state), the answer is the source itself when a start state is final
(engine.py:154-160).  Same results as the device run, for every algorithm, and
the device-side accessors still work afterwards."""

import ctypes
import json
import math
import os

import numpy as np
import pytest

import paper_2412_10287_b200 as P
from paper_2412_10287_b200 import _lib, datagen

pytestmark = pytest.mark.gpu

AUTOS = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "extra_automata.json")))


def _no_seed_edge_sources(sg, n, count=6):
    """Vertices without an out-edge (in-edge for inverted symbols) in any symbol a start state reads."""
    has = np.zeros(sg.nv, dtype=bool)
    for (idx, inverted), m in n.transitions.items():
        rows = np.asarray(m.indptr)
        if idx >= sg.nl or not any(rows[q + 1] > rows[q] for q in n.start_set):
            continue
        ends = sg.dst if inverted else sg.src
        has[ends[sg.lab == idx]] = True
    return [int(v) for v in np.flatnonzero(~has)[:count]], [int(v) for v in np.flatnonzero(has)[:2]]


@pytest.mark.parametrize("query", ["a ^b* c", "(a|^b)* c+", "(a b)* | (c ^d)+ e?"])
def test_host_answered_matches_device(query):
    from oracle import OracleGraph, OracleQuery, oracle_bfs

    sg = datagen.gen_rmat(12, 4, 8, 1.0, 23)
    g = sg.labeled_graph()
    og = OracleGraph(sg.nv, sg.nl, sg.src, sg.dst, sg.lab)
    nj = AUTOS[query]
    n = P.Automaton.from_json(nj)
    oq = OracleQuery(nj, sg.nl)
    empty, busy = _no_seed_edge_sources(sg, n)
    assert empty
    for s in empty + busy:
        want, st = oracle_bfs(og, oq, s)
        for algorithm in ("hybrid", "masked", "no_mask"):
            fast = P.eval_ssr(g, n, s, P.EngineOptions(timeout=math.inf, algorithm=algorithm))
            dev = P.eval_ssr(g, n, s, P.EngineOptions(timeout=math.inf, algorithm=algorithm, count_te=True))
            assert np.array_equal(fast.reach, want) and np.array_equal(dev.reach, want), (s, algorithm)
            assert fast.iterations == dev.iterations == st["iterations"], (s, algorithm)
            assert fast.reachable == dev.reachable
        # debug mode (device-side invariants) right after a host-answered call
        P.eval_ssr(g, n, s, P.EngineOptions(timeout=math.inf))
        chk = P.eval_ssr(g, n, s, P.EngineOptions(timeout=math.inf, debug_checks=True))
        assert np.array_equal(chk.reach, want)


def test_device_accessors_after_a_host_answered_call():
    sg = datagen.gen_rmat(12, 4, 8, 1.0, 23)
    g = sg.labeled_graph()
    n = P.Automaton.from_json(AUTOS["a ^b* c"])
    empty, _ = _no_seed_edge_sources(sg, n)
    s = empty[0]
    lib = _lib.engine()
    pq = P.PreparedQuery(g, n)
    try:
        st = _lib.RpqStats()
        nwords = (sg.nv + 31) // 32
        words = np.full(nwords, 0xFFFFFFFF, dtype=np.uint32)
        assert lib.rpq_query_eval(pq.q, s, -1.0, 0, 0, 4.0, 1, ctypes.addressof(st), words.ctypes.data, nwords) == 0
        assert st.grid == 0 and st.iterations == 1 and not words.any()  # answered on the host
        visited = np.zeros(nwords * n.nstates, dtype=np.uint32)
        assert lib.rpq_query_copy_visited(pq.q, _lib.ptr(visited, ctypes.c_uint32), visited.size) == 0
        assert int(np.unpackbits(visited.view(np.uint8)).sum()) == len(n.start_set)  # P = the seed, from the device
        reach = np.ones(sg.nv, dtype=np.uint8)
        assert lib.rpq_query_copy_reach(pq.q, _lib.ptr(reach, ctypes.c_uint8)) == 0
        assert not reach.any()
    finally:
        pq.close()
