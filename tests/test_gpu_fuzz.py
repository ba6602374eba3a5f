"""Randomised parity sweep: R-MAT and Erdos-Renyi graphs of assorted sizes
and skews, every extra automaton shape, hub and random sources, under every
direction policy and both kernels -- answers, iteration counts, TE and |P|
against the oracle.  Exercises the paths the fixed cases hit rarely: deferred
emission, seed bundles over many warps, hub rows, plan epochs after pulls."""

import json
import math
import os

import numpy as np
import pytest

from fixtures import automaton

import paper_2412_10287_b200 as P
from paper_2412_10287_b200 import datagen

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _er(nv, ne, nl, seed):
    rng = np.random.default_rng(seed)
    src = rng.integers(0, nv, ne).astype(np.int32)
    dst = rng.integers(0, nv, ne).astype(np.int32)
    lab = rng.integers(0, nl, ne).astype(np.int32)
    return nv, nl, src, dst, lab


@pytest.mark.parametrize("seed", range(8))
def test_fuzz_vs_oracle(seed):
    from oracle import OracleGraph, OracleQuery, oracle_bfs

    rng = np.random.default_rng(1000 + seed)
    autos = json.load(open(os.path.join(GOLDEN, "extra_automata.json")))
    if seed % 2 == 0:
        sg = datagen.gen_rmat(int(rng.integers(11, 19)), int(rng.integers(4, 20)), 8,
                              float(rng.uniform(0.5, 1.5)), 2000 + seed)
        nv, nl, src, dst, lab = sg.nv, sg.nl, sg.src, sg.dst, sg.lab
    else:
        nv, nl, src, dst, lab = _er(int(rng.integers(2000, 500000)), int(rng.integers(5000, 4000000)), 6,
                                    3000 + seed)
    g = P.LabeledGraph.from_coo(nv, [chr(ord("a") + i) for i in range(nl)], src, dst, lab)
    og = OracleGraph(nv, nl, src, dst, lab)
    deg = np.bincount(src, minlength=nv)
    sources = [int(np.argmax(deg)), int(rng.integers(0, nv)), int(rng.integers(0, nv))]
    evals = 0
    for query in sorted(autos):
        nj = autos[query]
        n = automaton(nj)
        oq = OracleQuery(nj, nl)
        for s in sources:
            want, st = oracle_bfs(og, oq, s)
            for direction, kernel in (("auto", "auto"), ("push", "grid"), ("pull", "grid"), ("auto", "grid")):
                got = P.eval_ssr(g, n, s, P.EngineOptions(timeout=math.inf, direction=direction, kernel=kernel,
                                                          algorithm="masked", count_te=True))
                assert np.array_equal(got.reach, want), (seed, query, s, direction, kernel)
                assert got.iterations == st["iterations"], (seed, query, s, direction, kernel)
                assert got.stats["te"] == st["te"], (seed, query, s, direction, kernel)
                assert got.stats["visited_pairs"] == st["pairs"], (seed, query, s, direction, kernel)
                evals += 1
        # the batch kernel on the same sources
        rows = P.eval_ssr_batch(g, n, sources, P.EngineOptions(timeout=math.inf))
        for i, s in enumerate(sources):
            assert np.array_equal(rows[i], oracle_bfs(og, oq, s)[0]), (seed, query, s, "batch")
    assert evals == 12 * len(autos)
