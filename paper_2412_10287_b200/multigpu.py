"""Multi-GPU plumbing for independent single-source queries (one process per
GPU, torch.distributed for the plumbing only).

The reference evaluates one query per call on one CPU thread; its bench runs
independent workload entries on a thread pool (rpq/cli.py:136-139).  Here
independent queries (sources) are sharded across ranks with no data-path
collective: every rank holds a replica of the graph and evaluates its own
sources ("replicas").  The only collectives are the
measurement's: the max over ranks of the device time and the sum of the
product edges traversed.
"""

import torch
import torch.distributed as dist


def shard(items, rank, world):
    """The items rank `rank` of `world` evaluates (round-robin, stable)."""
    return [x for i, x in enumerate(items) if i % world == rank]


def ranked_sources(out_degree, k):
    """The k vertices of highest out-degree (ties: lowest id) -- rank r of a
    weak-scaling run starts its query from the r-th."""
    import numpy as np

    order = np.lexsort((np.arange(out_degree.size), -out_degree))
    return [int(v) for v in order[:k]]


def reduce_timing(total_ms, units, device=None):
    """(max over ranks of total_ms, sum over ranks of units).  A no-op on one
    process; uses whatever backend the process group was created with (NCCL on
    the GPU box, gloo in the CPU tests)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(total_ms), float(units)
    dev = device if device is not None else torch.device("cpu")
    t = torch.tensor([float(total_ms)], dtype=torch.float64, device=dev)
    u = torch.tensor([float(units)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(u, op=dist.ReduceOp.SUM)
    return float(t.item()), float(u.item())
