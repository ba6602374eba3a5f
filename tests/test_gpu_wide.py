"""Automata beyond the persistent kernel's table limits (more than 256 states
or (state, symbol) groups, more than 128 symbols): eval_ssr falls back to
rpq_ssr_wide.  The reference has no such limit (engine.py:99-102 iterates
N.alphabet), so these must evaluate -- and bit-exactly: answers and iteration
counts against the CPU oracle, for every algorithm."""

import math

import numpy as np
import pytest

import paper_2412_10287_b200 as P
from paper_2412_10287_b200 import datagen, engine
from paper_2412_10287_b200.automaton import transition_table

pytestmark = pytest.mark.gpu


def _random_automaton(rng, nstates, symbols, ntrans, nstarts=2, nfinals=5):
    trans = {}
    for _ in range(ntrans):
        sym = symbols[int(rng.integers(len(symbols)))]
        trans.setdefault(sym, set()).add((int(rng.integers(nstates)), int(rng.integers(nstates))))
    return {
        "nstates": nstates,
        "transitions": [[s[0], s[1], sorted(list(p) for p in pairs)] for s, pairs in sorted(trans.items())],
        "alphabet": sorted([list(s) for s in trans]),
        "starts": sorted(int(x) for x in rng.choice(nstates, size=nstarts, replace=False)),
        "finals": sorted(int(x) for x in rng.choice(nstates, size=nfinals, replace=False)),
    }


def _check(sg, nj, sources):
    from oracle import OracleGraph, OracleQuery, oracle_bfs

    g = sg.labeled_graph()
    og = OracleGraph(sg.nv, sg.nl, sg.src, sg.dst, sg.lab)
    n = P.Automaton.from_json(nj)
    assert engine._is_wide(transition_table(n, sg.nl))
    oq = OracleQuery(nj, sg.nl)
    for s in sources:
        want, st = oracle_bfs(og, oq, s)
        for algorithm in ("hybrid", "masked", "no_mask"):
            got = P.eval_ssr(g, n, s, P.EngineOptions(timeout=math.inf, algorithm=algorithm, count_te=True))
            assert np.array_equal(got.reach, want), (s, algorithm)
            assert got.iterations == st["iterations"], (s, algorithm)
            assert got.stats["visited_pairs"] == st["pairs"]
            assert got.stats["te"] == st["te"]
    return g, n


def test_more_than_256_states():
    rng = np.random.default_rng(0x57A7E5)
    sg = datagen.gen_rmat(11, 8, 4, 1.0, 7)
    symbols = [(l, inv) for l in range(4) for inv in (False, True)]
    nj = _random_automaton(rng, 700, symbols, 2500)
    _check(sg, nj, [0, 5, int(np.argmax(sg.out_degree())), sg.nv - 1])


def test_more_than_128_symbols():
    rng = np.random.default_rng(0x5B01)
    sg = datagen.gen_rmat(10, 16, 80, 0.5, 11)
    symbols = [(l, inv) for l in range(80) for inv in (False, True)]  # 160 symbols
    nj = _random_automaton(rng, 40, symbols, 1200)
    assert len(nj["alphabet"]) > 128
    _check(sg, nj, [0, 1, 2, int(np.argmax(sg.out_degree()))])


def test_more_than_256_groups():
    rng = np.random.default_rng(0x6209)
    sg = datagen.gen_rmat(10, 8, 6, 1.0, 13)
    symbols = [(l, inv) for l in range(6) for inv in (False, True)]
    nj = _random_automaton(rng, 200, symbols, 1500)
    g, n = _check(sg, nj, [3, int(np.argmax(sg.out_degree()))])
    # an empty start set and the reference's timeout rule go through the same path
    nj2 = dict(nj, starts=[])
    n2 = P.Automaton.from_json(nj2)
    assert P.eval_ssr(g, n2, 0, P.EngineOptions(algorithm="masked")).iterations == 0
    assert P.eval_ssr(g, n2, 0, P.EngineOptions(algorithm="hybrid")).iterations == 1
    with pytest.raises(P.QueryTimeout):
        P.eval_ssr(g, n, 3, P.EngineOptions(timeout=0.0))
    # SDR is SSR on the reversed automaton: wide as well
    back = P.eval_sdr(g, n, 3, P.EngineOptions(timeout=math.inf))
    assert back.iterations >= 1
