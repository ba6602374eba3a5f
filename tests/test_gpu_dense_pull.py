"""Pull levels whose 1,024-vertex tasks hold more candidates than the per-warp
queue (768 vertex ids): a dense Erdos-Renyi graph, large enough for the
large-graph task size (>= 2.4M vertices), pulled from the first level on, when
nearly every vertex is unvisited and has in-edges.  Both variants: targets with
one in-slot (straight-line pull) and with several (step loop).  Against the
oracle, bit-exact, with exact |P| and TE."""

import math

import numpy as np
import pytest

import paper_2412_10287_b200 as P
from paper_2412_10287_b200 import datagen

pytestmark = pytest.mark.gpu


def _nfa(nstates, trans, starts, finals):
    return {"nstates": nstates,
            "transitions": [[l, inv, pairs] for (l, inv), pairs in sorted(trans.items())],
            "alphabet": sorted([[l, inv] for (l, inv) in trans]),
            "starts": starts, "finals": finals}


@pytest.fixture(scope="module")
def dense():
    from oracle import OracleGraph

    sg = datagen.gen_er(2_600_000, 40_000_000, 2, 0xD5E)
    return sg, sg.labeled_graph(), OracleGraph(sg.nv, sg.nl, sg.src, sg.dst, sg.lab)


@pytest.mark.parametrize("name,nj", [
    # a*: one state, one in-slot
    ("a*", _nfa(1, {(0, False): [[0, 0]]}, [0], [0])),
    # (a | b b)*: state 0 is entered by a (from 0) and by b (from 1): two in-slots
    ("(a|b b)*", _nfa(2, {(0, False): [[0, 0]], (1, False): [[0, 1], [1, 0]]}, [0], [0])),
    # a ^b*: an inverted symbol, a target entered from two states by the same symbol
    ("a ^b*", _nfa(2, {(0, False): [[0, 1]], (1, True): [[1, 1]]}, [0], [1])),
    # a b a a*: four states (|Q| x |V| >= 8M pairs: the 1,024-thread kernel instance)
    ("a b a a*", _nfa(4, {(0, False): [[0, 1], [2, 3], [3, 3]], (1, False): [[1, 2]]}, [0], [3])),
])
def test_dense_first_pull_level(dense, name, nj):
    from oracle import OracleQuery, oracle_bfs

    sg, g, og = dense
    n = P.Automaton.from_json(nj)
    oq = OracleQuery(nj, sg.nl)
    for s in (0, 1_234_567):
        want, st = oracle_bfs(og, oq, s)
        for direction in ("pull", "auto"):
            got = P.eval_ssr(g, n, s, P.EngineOptions(timeout=math.inf, direction=direction, count_te=True,
                                                      kernel="grid"))
            assert np.array_equal(got.reach, want), (name, s, direction)
            assert got.iterations == st["iterations"], (name, s, direction)
            assert got.stats["visited_pairs"] == st["pairs"] and got.stats["te"] == st["te"]
