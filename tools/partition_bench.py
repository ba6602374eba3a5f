"""Vertex-partitioned single query (SURVEY.md §8(e) regime 2), cfg3 by default.

    # k ranks, one GPU each (NCCL allgather of frontier slices every level)
    python -m torch.distributed.run --nproc-per-node K --master-addr 127.0.0.1 \\
        tools/partition_bench.py [--config cfg3] [--reps 3]
    # k shards in ONE process on one GPU (sequential; per-shard step time only)
    python tools/partition_bench.py --local-shards K

Prints one JSON line: query time (wall, max over ranks), GTEPS over the
query's exact TE, levels, and per level the max over shards of the step
kernel's device time -- the compute part of the sharded roofline."""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--local-shards", type=int, default=0)
    args = ap.parse_args()

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2412_10287_b200 as P
    from paper_2412_10287_b200 import datagen, partition
    from paper_2412_10287_b200.automaton import transition_table

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    distributed = world > 1 or "RANK" in os.environ
    if distributed:
        dist.init_process_group("nccl", device_id=dev)
    autos = json.load(open(os.path.join(ROOT, "paper_2412_10287_b200", "data", "config_automata.json")))
    c = datagen.CONFIGS[args.config]
    query = c["queries"][0]
    n = P.Automaton.from_json(autos[args.config][f"{query}|min"])
    sg = datagen.generate(args.config)
    g = sg.labeled_graph()
    source = int(datagen.pick_sources(sg, args.config, count=1)[0])
    table = transition_table(n, g.num_labels)
    k = args.local_shards or world
    ranges = partition.partition_words(partition.target_weights(g, table), k)
    t = time.time()
    if args.local_shards:
        shards = [partition.Shard(g, n, ranges, r, dev) for r in range(k)]
        ex = partition.LocalExchange()
    else:
        shards = [partition.Shard(g, n, ranges, rank, dev)]
        ex = partition.DistExchange()
    build_s = time.time() - t
    # exact TE of this query (single-GPU engine, count_te) for the GTEPS figure
    te = None
    if rank == 0:
        pq = P.PreparedQuery(g, n)
        pq.set_options(count_te=True)
        pq.launch(source)
        st = pq.wait()
        te = int(st.te)
        want = pq.reach()
        want_bits = np.packbits(want, bitorder="little").view(np.uint8)
        single_ms = []
        pq.set_options(count_te=False)
        for _ in range(args.reps):
            pq.launch(source)
            single_ms.append(pq.wait().device_ms)
        pq.close()
    args_run = (shards, ex, ranges, g.num_vertices, table.starts.tolist(), table.finals.tolist(), source)
    reach0, its0, prof = partition.run_levels(*args_run, profile=True)  # warm-up + per-level step times
    bits0 = None
    partition.run_levels(*args_run, bits=True)  # second warm-up (first runs allocate and touch memory)
    walls = []
    for _ in range(args.reps):
        if distributed:
            dist.barrier()
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        words, its, _ = partition.run_levels(*args_run, bits=True)
        torch.cuda.synchronize(dev)
        walls.append(time.perf_counter() - t0)
    wall = float(np.median(walls))
    if distributed:
        tt = torch.tensor([wall], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        wall = float(tt.item())
    if rank == 0:
        per_level_max = [max(x) for x in prof["step_ms"]]
        out = {
            "mode": "local-shards" if args.local_shards else "ranks", "k": k, "config": args.config,
            "query": query, "source": source, "vertices": sg.nv, "edges": sg.ne,
            "iterations": its,
            "parity_vs_single_gpu": bool(np.array_equal(words.view(np.uint8)[: want_bits.size], want_bits)),
            "profile_run": {"iterations": its0, "parity": bool(np.array_equal(reach0, want)),
                            "levels_wall_us": prof["levels_wall_us"]},
            "te": te, "query_ms_wall": 1e3 * wall,
            "gteps_wall": te / wall / 1e9 if te else None,
            "step_ms_max_over_shards": per_level_max, "step_ms_sum": sum(per_level_max),
            "single_gpu_fused_ms": float(np.median(single_ms)),
            "ranges_words": ranges, "build_s": build_s,
        }
        print(json.dumps(out), flush=True)
    for sh in shards:
        sh.step.close()
    if distributed:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
