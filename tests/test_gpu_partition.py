"""Vertex-partitioned evaluation (SURVEY.md §8(e) regime 2) on the device:
k shards -- each with its own rank graph (edges whose traversal target it
owns) and its own step kernel -- run in one process on one GPU, exchanging
frontier slices by a stack instead of NCCL (no shard waits on another).  The
answer and the masked iteration count must equal the oracle's for every k."""

import json
import math
import os

import numpy as np
import pytest
import torch

from fixtures import automaton, unpack_bits
from conftest import load_golden

import paper_2412_10287_b200 as P
from paper_2412_10287_b200 import datagen, partition
from paper_2412_10287_b200.automaton import transition_table

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _run_local(g, n, source, k):
    table = transition_table(n, g.num_labels)
    ranges = partition.partition_words(partition.target_weights(g, table), k)
    dev = torch.device("cuda", 0)
    shards = [partition.Shard(g, n, ranges, r, dev) for r in range(k)]
    try:
        return partition.run_levels(shards, partition.LocalExchange(), ranges, g.num_vertices,
                                    table.starts.tolist(), table.finals.tolist(), source)
    finally:
        for sh in shards:
            sh.step.close()


@pytest.mark.parametrize("k", [1, 2, 3, 8])
@pytest.mark.parametrize("scale,seed,query", [
    (14, 21, "^a (b|c)* d"), (15, 22, "a ^b* c"), (13, 24, "(a|^b)* c+"),
    (12, 25, "(a ^a)* (b | c ^d)*"), (13, 27, "a ^b c*")])
def test_partitioned_vs_oracle(scale, seed, query, k):
    from oracle import OracleGraph, OracleQuery, oracle_bfs

    sg = datagen.gen_rmat(scale, 16, 8, 1.0, seed)
    g = sg.labeled_graph()
    og = OracleGraph(sg.nv, sg.nl, sg.src, sg.dst, sg.lab)
    nj = json.load(open(os.path.join(GOLDEN, "extra_automata.json")))[query]
    n = automaton(nj)
    oq = OracleQuery(nj, sg.nl)
    deg = sg.out_degree()
    for s in (int(np.argmax(deg)), sg.nv - 1):
        want, st = oracle_bfs(og, oq, s)
        reach, its, _ = _run_local(g, n, s, k)
        assert np.array_equal(reach, want), (query, s, k)
        assert its == st["iterations"], (query, s, k)


def test_partitioned_cfg2_golden():
    gold = load_golden("cfg2.json.gz")
    sg = datagen.generate("cfg2")
    assert sg.digest() == gold["digest"]
    g = sg.labeled_graph()
    for rec in gold["records"][:2]:
        n = automaton(rec["nfa"])
        want = unpack_bits(rec["reach_bits"], sg.nv)
        for k in (2, 4):
            reach, its, _ = _run_local(g, n, rec["source"], k)
            assert np.array_equal(reach, want), k
            assert its == rec["iterations"]["masked"], k


def test_partition_edge_cases():
    n = P.Automaton.build(1, {(0, False): [(0, 0)]}, [0], [0])
    g = P.LabeledGraph.from_edges(5, ["a"], [(0, 0, 1), (1, 0, 2), (3, 0, 3)])
    for k in (1, 2, 4):
        reach, its, _ = _run_local(g, n, 0, k)
        assert reach.tolist() == [1, 1, 1, 0, 0] and its == 3
        reach, its, _ = _run_local(g, n, 4, k)
        assert reach.tolist() == [0, 0, 0, 0, 1] and its == 1


def test_first_step_after_create_keeps_p():
    """Regression: the kernel read its per-run arguments from shared memory
    before every thread could see them, so a query's first step-mode launch
    could run as a full evaluation (clearing P and M)."""
    sg = datagen.gen_rmat(16, 16, 8, 1.0, 77)
    g = sg.labeled_graph()
    nj = json.load(open(os.path.join(GOLDEN, "extra_automata.json")))["^a (b|c)* d"]
    n = automaton(nj)
    for _ in range(3):
        reach, its, _ = _run_local(g, n, int(np.argmax(sg.out_degree())), 1)
        want = P.eval_ssr(g, n, int(np.argmax(sg.out_degree())), P.EngineOptions(algorithm="masked"))
        assert np.array_equal(reach, want.reach) and its == want.iterations
