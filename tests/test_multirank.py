"""Multi-rank host logic on CPU: world_size 2 over gloo (127.0.0.1).

The data path has no collective (independent queries per rank, SURVEY.md
§8(e)); these tests cover what the bench does across ranks: disjoint and
complete source sharding, max-over-ranks time, summed units, and the oracle
answers each rank would check against."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2412_10287_b200 import multigpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, results):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sources = list(range(10))
        mine = multigpu.shard(sources, rank, world)
        # each rank "times" its shard: 1 ms per source plus a rank skew
        total_ms = 1.0 * len(mine) + 0.5 * rank
        units = 100 * len(mine)
        t, u = multigpu.reduce_timing(total_ms, units)
        results[rank] = (mine, t, u)
    finally:
        dist.destroy_process_group()


def test_shard_and_reduce_two_ranks():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, port, results), nprocs=world, join=True)
    mine0, t0, u0 = results[0]
    mine1, t1, u1 = results[1]
    assert sorted(mine0 + mine1) == list(range(10)) and not set(mine0) & set(mine1)
    assert t0 == t1 == max(1.0 * len(mine0), 1.0 * len(mine1) + 0.5)
    assert u0 == u1 == 1000


def test_single_process_reduce_is_identity():
    assert multigpu.reduce_timing(3.5, 7) == (3.5, 7.0)


def test_ranked_sources_ties_lowest_id():
    deg = np.array([3, 5, 5, 1, 5])
    assert multigpu.ranked_sources(deg, 4) == [1, 2, 4, 0]


def test_rank_sources_have_oracle_answers():
    """Every rank's query has a well-defined CPU answer (the checker each
    rank would use), independent of how the sources were sharded."""
    import json
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.join(root, "oracle"))
    from oracle import OracleGraph, OracleQuery, oracle_bfs

    from paper_2412_10287_b200 import datagen

    sg = datagen.gen_rmat(12, 16, 8, 1.0, seed=31)
    og = OracleGraph(sg.nv, sg.nl, sg.src, sg.dst, sg.lab)
    nj = json.load(open(os.path.join(root, "tests", "golden", "extra_automata.json")))["a ^b* c"]
    oq = OracleQuery(nj, sg.nl)
    srcs = multigpu.ranked_sources(sg.out_degree(), 4)
    per_rank = [multigpu.shard(srcs, r, 2) for r in range(2)]
    answers = {s: oracle_bfs(og, oq, s)[0] for r in per_rank for s in r}
    assert set(answers) == set(srcs)
    assert all(a.dtype == np.uint8 and a.size == sg.nv for a in answers.values())


# ---- vertex-partitioned single query (SURVEY.md §8(e) regime 2) -----------


def _partition_worker(rank, world, port, results):
    import json
    import sys

    import torch
    import torch.distributed as dist

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.join(root, "tests"))
    from partition_helpers import CpuStep

    from paper_2412_10287_b200 import datagen, partition
    from paper_2412_10287_b200.automaton import Automaton, transition_table

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        autos = json.load(open(os.path.join(root, "tests", "golden", "extra_automata.json")))
        out = {}
        for query, seed in (("a ^b* c", 41), ("(a|^b)* c+", 42), ("^a (b|c)* d", 43)):
            sg = datagen.gen_rmat(10, 8, 6, 1.0, seed)
            g = sg.labeled_graph()
            n = Automaton.from_json(autos[query])
            table = transition_table(n, g.num_labels)
            ranges = partition.partition_words(partition.target_weights(g, table), world)
            w0, w1 = ranges[rank]
            lg, ln = partition.local_problem(g, n, min(32 * w0, g.num_vertices), min(32 * w1, g.num_vertices))
            sh = partition.Shard(g, n, ranges, rank, torch.device("cpu"), step=CpuStep(lg, ln, g.num_vertices))
            ex = partition.DistExchange()
            src = int(np.argmax(sg.out_degree()))
            reach, its, _ = partition.run_levels([sh], ex, ranges, g.num_vertices, table.starts.tolist(),
                                                 table.finals.tolist(), src)
            out[query] = (reach.tolist(), its, ranges, src, seed)
        results[rank] = out
    finally:
        dist.destroy_process_group()


def test_partitioned_two_ranks_match_oracle():
    """Two gloo ranks, each owning half of the vertices (balanced by target
    degree), exchange frontier slices every level; both end with the oracle's
    answer and the masked loop's iteration count."""
    import json
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.join(root, "oracle"))
    from oracle import OracleGraph, OracleQuery, oracle_bfs

    from paper_2412_10287_b200 import datagen

    world = 2
    port = _free_port()
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_partition_worker, args=(world, port, results), nprocs=world, join=True)
    autos = json.load(open(os.path.join(root, "tests", "golden", "extra_automata.json")))
    for query, (reach, its, ranges, src, seed) in results[0].items():
        assert results[1][query][0] == reach and results[1][query][1] == its
        assert ranges[0][0] == 0 and ranges[0][1] == ranges[1][0] and 0 < ranges[0][1] < ranges[1][1]
        sg = datagen.gen_rmat(10, 8, 6, 1.0, seed)
        og = OracleGraph(sg.nv, sg.nl, sg.src, sg.dst, sg.lab)
        want, st = oracle_bfs(og, OracleQuery(autos[query], sg.nl), src)
        assert np.array_equal(np.array(reach, dtype=np.uint8), want), query
        assert its == st["iterations"], query


def test_partition_ranges_balanced():
    from paper_2412_10287_b200 import partition

    w = np.array([100, 1, 1, 1, 1, 1, 1, 1, 1, 100], dtype=np.int64)
    r = partition.partition_words(w, 2)
    assert r == [(0, 5), (5, 10)]
    r = partition.partition_words(np.ones(3, dtype=np.int64), 5)
    assert r[0][0] == 0 and r[-1][1] == 3 and all(a <= b for a, b in r)
    assert sum(b - a for a, b in r) == 3
