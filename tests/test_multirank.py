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
