"""Vertex-partitioned evaluation of ONE single-source query across k GPUs
(regime 2; north_star: "partitions vertices 1-D across the
GPUs of one box and exchanges frontier bitmaps each level with NCCL
allgather").

Partition.  Vertices are cut into k contiguous ranges of whole 32-vertex
words, balanced by the work a range receives: per vertex 1 + the number of
product edges that can land on it (in-degree over the labels the query reads
forward, out-degree over the labels it reads inverted).

Per-rank graph.  Rank r keeps only the edges whose TRAVERSAL TARGET is in its
range: for a forward symbol l the edges (u -l-> v) with v in range, for an
inverted symbol l the edges with u in range.  The two subsets differ, so they
are stored as two labels of the rank's graph (2l for forward use, 2l+1 for
inverted use) and the automaton is relabelled to match; the step kernel then
expands the full frontier and can only discover pairs in its own range.

Per level (the masked loop, engine.py:146-171):
    every rank:  next_r = step(M) <not P_r>;  P_r |= next_r     (one kernel)
    all ranks:   M = allgather(next_r restricted to range r)   (one collective)
    every rank:  stop when M is empty (identical on all ranks: no extra
                 collective)
The frontier M is replicated; P is meaningful on the owned range only.  The
answer is the allgather of every rank's OR over final states.

The step is the persistent kernel in step mode (push only) through
``rpq_query_step_device``; the exchange is ``torch.distributed`` (NCCL on the
GPU box, gloo in the CPU tests).  ``LocalExchange`` runs k shards in one
process (sequentially, no cross-shard waiting) to test the partitioned path on
one GPU.
"""

import ctypes
import math
import time

import numpy as np

from . import _lib
from .automaton import Automaton, _matrix_pairs, transition_table


# ---------------------------------------------------------------------------
# partition
# ---------------------------------------------------------------------------


def _coo(g):
    """(src, dst, lab) int32 arrays of a host graph (its edge list if it was
    built from one, else read back from the per-label CSR)."""
    coo = getattr(g, "_coo", None)
    if coo is not None:
        return coo
    src, dst, lab = [], [], []
    for l in range(g.num_labels):
        m = g.forward[l]
        rows = np.repeat(np.arange(m.nrows, dtype=np.int64), np.diff(np.asarray(m.indptr)))
        src.append(rows.astype(np.int32))
        dst.append(np.asarray(m.indices, dtype=np.int32))
        lab.append(np.full(rows.size, l, dtype=np.int32))
    cat = (lambda xs: np.concatenate(xs) if xs else np.zeros(0, np.int32))
    return cat(src), cat(dst), cat(lab)


def _uses(table):
    """{label: (read forward, read inverted)} of the query's usable symbols."""
    out = {}
    for l, inv in zip(table.t_label.tolist(), table.t_inv.tolist()):
        f, b = out.get(l, (False, False))
        out[l] = (f or not inv, b or bool(inv))
    return out


def target_weights(g, table):
    """Per 32-vertex word: 32 + the product edges whose target lies in it."""
    nv = int(g.num_vertices)
    src, dst, lab = _coo(g)
    w = np.ones(nv, dtype=np.int64)
    for l, (fwd, inv) in _uses(table).items():
        sel = lab == l
        if fwd:
            w += np.bincount(dst[sel], minlength=nv)
        if inv:
            w += np.bincount(src[sel], minlength=nv)
    nwords = (nv + 31) // 32
    pad = np.zeros(nwords * 32, dtype=np.int64)
    pad[:nv] = w
    return pad.reshape(nwords, 32).sum(axis=1)


def partition_words(word_weights, k):
    """k contiguous word ranges [(w0, w1)) of near-equal weight (empty ranges
    allowed when there are fewer words than ranks)."""
    k = int(k)
    nwords = int(word_weights.size)
    if k < 1:
        raise ValueError("k must be >= 1")
    cum = np.concatenate([[0], np.cumsum(word_weights)])
    total = cum[-1]
    cuts = [0]
    for r in range(1, k):
        c = int(np.searchsorted(cum, total * r / k, side="left"))
        cuts.append(min(max(c, cuts[-1]), nwords))
    cuts.append(nwords)
    return [(cuts[r], cuts[r + 1]) for r in range(k)]


def local_problem(g, n, v0, v1):
    """(graph, automaton) of the rank owning vertices [v0, v1): edges whose
    traversal target is in the range, forward uses relabelled 2l, inverted
    uses 2l+1."""
    from .graph import LabeledGraph

    table = transition_table(n, g.num_labels)
    src, dst, lab = _coo(g)
    ls, ld, ll = [], [], []
    for l, (fwd, inv) in _uses(table).items():
        sel = lab == l
        s, d = src[sel], dst[sel]
        if fwd:
            m = (d >= v0) & (d < v1)
            ls.append(s[m]), ld.append(d[m]), ll.append(np.full(int(m.sum()), 2 * l, np.int32))
        if inv:
            m = (s >= v0) & (s < v1)
            ls.append(s[m]), ld.append(d[m]), ll.append(np.full(int(m.sum()), 2 * l + 1, np.int32))
    cat = (lambda xs: np.concatenate(xs).astype(np.int32) if xs else np.zeros(0, np.int32))
    names = [f"{i // 2}{'^' if i % 2 else ''}" for i in range(2 * g.num_labels)]
    lg = LabeledGraph.from_coo(g.num_vertices, names, cat(ls), cat(ld), cat(ll))
    trans = {}
    for idx, inverted in sorted(n.alphabet):
        if not 0 <= idx < g.num_labels:  # engine.py:100-101
            continue
        rows, cols = _matrix_pairs(n.transitions[(idx, inverted)])
        trans[(2 * idx + int(inverted), inverted)] = list(zip(rows.tolist(), cols.tolist()))
    ln = Automaton.build(n.nstates, trans, sorted(n.start_set), sorted(n.final_set))
    return lg, ln


# ---------------------------------------------------------------------------
# exchange
# ---------------------------------------------------------------------------


class DistExchange:
    """allgather over the default torch.distributed group (one shard per rank)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def allgather(self, slices):
        import torch

        (mine,) = slices
        out = torch.empty((self.world,) + tuple(mine.shape), dtype=mine.dtype, device=mine.device)
        if mine.is_cuda:
            self.dist.all_gather_into_tensor(out, mine.contiguous(), group=self.group)
        else:
            self.dist.all_gather(list(out.unbind(0)), mine.contiguous(), group=self.group)
        return out


class LocalExchange:
    """All k shards live in this process: the gather is a stack."""

    def allgather(self, slices):
        import torch

        return torch.stack([s.contiguous() for s in slices])


# ---------------------------------------------------------------------------
# shards and the level loop
# ---------------------------------------------------------------------------


class DeviceStep:
    """next = step(M) <not P>, P |= next: the persistent kernel's step mode on
    the rank's graph (rpq_query_step_device)."""

    def __init__(self, lg, ln, device, owned=None):
        from .engine import PreparedQuery

        from .engine import raise_for_status

        import torch

        self.pq = PreparedQuery(lg, ln, device=torch.device(device).index or 0)

        w = ctypes.c_int64()
        raise_for_status(_lib.engine().rpq_query_row_words(self.pq.q, ctypes.byref(w)), "rpq_query_row_words")
        self.row_words = int(w.value)
        if owned is not None:  # pull steps scan only the owned targets
            raise_for_status(_lib.engine().rpq_query_set_owned(self.pq.q, int(owned[0]), int(owned[1])),
                             "rpq_query_set_owned")

    def __call__(self, m, p, out, stream):
        from .engine import raise_for_status

        if not stream:
            raise ValueError("the step needs the caller's (non-default) CUDA stream")
        raise_for_status(_lib.engine().rpq_query_step_device(self.pq.q, m.data_ptr(), p.data_ptr(),
                                                             out.data_ptr(), stream), "rpq_query_step_device")

    def begin(self, stream):
        """Start a chain of steps on `stream` (zeroes the chain's counters)."""
        from .engine import raise_for_status

        raise_for_status(_lib.engine().rpq_query_step_begin(self.pq.q, stream), "rpq_query_step_begin")

    def count(self):
        """Wait for the chain so far: the steps whose M was non-empty (raises
        if any step of the chain failed)."""
        from .engine import raise_for_status

        n = ctypes.c_int64()
        raise_for_status(_lib.engine().rpq_query_step_end(self.pq.q, ctypes.byref(n)), "rpq_query_step_end")
        return int(n.value)

    def finish(self):
        """Status of the last step (raises on failure); its device time in ms."""
        from .engine import raise_for_status

        st = _lib.RpqStats()
        raise_for_status(_lib.engine().rpq_query_wait(self.pq.q, ctypes.byref(st)), "rpq_query_step_device")
        return float(st.device_ms)

    def close(self):
        self.pq.close()


class Shard:
    """One rank's share: owned word range, visited P, the step."""

    def __init__(self, g, n, ranges, r, device, step=None):
        import torch

        self.w0, self.w1 = ranges[r]
        nv = int(g.num_vertices)
        self.v0, self.v1 = min(32 * self.w0, nv), min(32 * self.w1, nv)
        self.nstates = int(n.nstates)
        self.device = device
        if step is None:
            lg, ln = local_problem(g, n, self.v0, self.v1)
            step = DeviceStep(lg, ln, device, owned=(self.w0, self.w1))
        self.step = step
        self.row_words = getattr(step, "row_words", ((nv + 31) // 32 + 3) // 4 * 4)
        shape = (self.nstates, self.row_words)
        self.p = torch.zeros(shape, dtype=torch.int32, device=device)
        self.next = torch.zeros(shape, dtype=torch.int32, device=device)


def _bit(v):
    return np.array([1 << (v & 31)], dtype=np.uint32).view(np.int32)[0].item()


def run_levels(shards, exchange, ranges, nv, starts, finals, source, timeout=math.inf, profile=False,
               bits=False):
    """The partitioned masked loop.  Returns (reach uint8[nv], iterations,
    stats) -- the answer as the uint32 bitmap instead with bits=True.  `shards`
    are the shards of THIS process (one per rank under torch.distributed, all k
    for LocalExchange).  Device work runs on one dedicated stream shared by the
    step kernels and the torch operations."""
    import contextlib

    import torch

    dev = shards[0].device
    if torch.device(dev).type == "cuda":
        s = getattr(shards[0], "stream", None)
        if s is None:  # one stream per shard set, reused across queries
            s = shards[0].stream = torch.cuda.Stream(dev)
        s.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(s):
            out = _run_levels(shards, exchange, ranges, nv, starts, finals, source, timeout, s.cuda_stream,
                              profile, bits)
        torch.cuda.current_stream(dev).wait_stream(s)
        return out
    return _run_levels(shards, exchange, ranges, nv, starts, finals, source, timeout, None, profile, bits)


def _run_levels(shards, exchange, ranges, nv, starts, finals, source, timeout, stream, profile, bits,
                depth=4):
    """The masked loop, `depth` levels enqueued per host check: each step
    counts (on the device) whether its M was non-empty, and once one finds M
    empty every later step does too (its output stays zero), so the host
    waits only once per `depth` levels and the iteration count is exact.
    profile=True checks after every level (per-level timings)."""
    import torch

    t0 = time.monotonic()
    dev = shards[0].device
    nstates = shards[0].nstates
    row_words = shards[0].row_words
    k = len(ranges)
    wmax = max(max(w1 - w0 for w0, w1 in ranges), 1)
    m = getattr(shards[0], "_m", None)
    if m is None or tuple(m.shape) != (nstates, row_words):
        m = torch.zeros((nstates, row_words), dtype=torch.int32, device=dev)
    else:
        m.zero_()
    # one shard owning everything: the step's output IS the next frontier (no exchange)
    alone = k == 1 and len(shards) == 1
    send = [torch.zeros((nstates, wmax), dtype=torch.int32, device=dev) for _ in shards] if not alone else []
    for sh in shards:
        sh.p.zero_()
    # seed M = P = {(q_s, source)} (engine.py:106-109, :154-155); P on its owner
    # (m and p are zero here: a fill of the one word is the OR, without the
    # gather / scatter kernels of an indexed update)
    sw, sb = source >> 5, _bit(source)
    for q in set(starts):
        m[q, sw: sw + 1].fill_(sb)
        for sh in shards:
            if sh.w0 <= sw < sh.w1:
                sh.p[q, sw: sw + 1].fill_(sb)
    counted = hasattr(shards[0].step, "count")
    if counted:
        for sh in shards:
            sh.step.begin(stream)
    levels_us = []
    step_ms = []  # profile: per level, each local shard's step kernel time
    sync = (lambda: torch.cuda.synchronize(dev)) if m.is_cuda else (lambda: None)
    if not counted or profile:
        depth = 1
    enqueued = 0
    iterations = 0
    while True:
        if not counted and not bool(m.any()):
            break
        if time.monotonic() - t0 > timeout:  # _Clock.check, engine.py:87-89
            from .engine import QueryTimeout

            raise QueryTimeout(time.monotonic() - t0, iterations)
        # (the first check after two levels: a source without a matching
        # out-edge -- half of cfg3's -- is done after its first step)
        for _ in range(min(depth, 2) if enqueued == 0 else depth):
            for sh in shards:
                sh.step(m, sh.p, sh.next, stream)
            enqueued += 1
            if alone:
                m, shards[0].next = shards[0].next, m  # the step zeroes its output first
            else:
                for sh, sl in zip(shards, send):
                    sl[:, : sh.w1 - sh.w0].copy_(sh.next[:, sh.w0: sh.w1])
                gathered = exchange.allgather(send)
                for r, (w0, w1) in enumerate(ranges):
                    m[:, w0:w1].copy_(gathered[r, :, : w1 - w0])
        if profile:
            sync()
            levels_us.append((time.monotonic() - t0) * 1e6)
            step_ms.append([sh.step.finish() if hasattr(sh.step, "finish") else 0.0 for sh in shards])
        if counted:
            iterations = shards[0].step.count()  # waits for the enqueued levels
            if iterations < enqueued:
                break
        else:
            iterations = enqueued
    shards[0]._m = m
    for sh in shards:
        if hasattr(sh.step, "finish"):
            sh.step.finish()
    if profile:
        levels_us = levels_us[: iterations + 1]
        step_ms = step_ms[: iterations + 1]
    # answer: OR over final states of each owner's P, gathered
    slices = []
    for sh in shards:
        sl = torch.zeros((1, wmax), dtype=torch.int32, device=dev)
        fl = sorted(set(finals))
        if fl:
            acc = sh.p[fl[0]: fl[0] + 1, sh.w0: sh.w1]
            if len(fl) > 1:
                acc = acc.clone()
                for f in fl[1:]:
                    acc |= sh.p[f: f + 1, sh.w0: sh.w1]
            sl[:, : sh.w1 - sh.w0] = acc
        slices.append(sl)
    gathered = exchange.allgather(slices)
    words = np.zeros(max(row_words, 1), dtype=np.uint32)
    if gathered.is_cuda:
        # a pinned staging buffer, kept with the shard set (a pageable copy of
        # cfg3's 2 MB answer costs more than the query's device time)
        host = getattr(shards[0], "_host", None)
        if host is None or host.shape != gathered.shape:
            host = shards[0]._host = torch.empty(gathered.shape, dtype=gathered.dtype, pin_memory=True)
        host.copy_(gathered, non_blocking=True)
        torch.cuda.current_stream(dev).synchronize()
        g_host = host.numpy().view(np.uint32)
    else:
        g_host = gathered.cpu().numpy().view(np.uint32)
    for r, (w0, w1) in enumerate(ranges):
        words[w0:w1] = g_host[r, 0, : w1 - w0]
    stats = {"levels_wall_us": levels_us, "ranges": ranges, "step_ms": step_ms, "enqueued": enqueued}
    if bits:
        return words, iterations, stats
    return np.unpackbits(words.view(np.uint8), bitorder="little")[:nv], iterations, stats


class PartitionedQuery:
    """One automaton on a vertex-partitioned graph, evaluated from many
    sources: the partition, this rank's graph (upload + device CSR/CSC), its
    step kernel and the bitmaps are built once.  One shard per
    torch.distributed rank (device = the rank's current CUDA device)."""

    def __init__(self, g, n, group=None, device=None):
        import torch

        self.g, self.n = g, n
        self.exchange = DistExchange(group)
        self.table = transition_table(n, g.num_labels)
        self.ranges = partition_words(target_weights(g, self.table), self.exchange.world)
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.shard = Shard(g, n, self.ranges, self.exchange.rank, dev)

    def run(self, source, timeout=math.inf, profile=False):
        """(answer bitmap words, masked-loop iterations, stats)."""
        return run_levels([self.shard], self.exchange, self.ranges, self.g.num_vertices,
                          self.table.starts.tolist(), self.table.finals.tolist(), int(source), timeout,
                          profile=profile, bits=True)

    def close(self):
        if self.shard is not None:
            self.shard.step.close()
            self.shard = None


_PARTITIONED = {}  # (id(g), id(n), group, world, rank, device) -> (weakrefs, PartitionedQuery)


def partitioned_query(g, n, group=None):
    """The cached PartitionedQuery of (g, n) on this rank (graphs and compiled
    automata are not mutated after construction; the entry dies with them)."""
    import weakref

    import torch.distributed as dist
    import torch

    key = (id(g), id(n), id(group), dist.get_world_size(group), dist.get_rank(group), torch.cuda.current_device())
    hit = _PARTITIONED.get(key)
    if hit is not None and hit[0]() is g and hit[1]() is n:
        return hit[2]
    pq = PartitionedQuery(g, n, group)
    try:
        refs = (weakref.ref(g, lambda _r, k=key: _drop(k)), weakref.ref(n, lambda _r, k=key: _drop(k)))
    except TypeError:
        return pq
    _PARTITIONED[key] = (refs[0], refs[1], pq)
    return pq


def _drop(key):
    hit = _PARTITIONED.pop(key, None)
    if hit is not None:
        hit[2].close()


def eval_ssr_partitioned(g, n, source, opts=None, group=None):
    """eval_ssr over vertex-partitioned ranks: one shard per torch.distributed
    rank (device = the rank's current CUDA device).  Returns the same
    EvalResult as eval_ssr: the caller's algorithm tag and that algorithm's
    iteration count (engine._iterations_for of the masked count)."""
    from .engine import _SSR_EVALUATORS, EngineOptions, EvalResult, QueryTimeout, _check_vertex, _iterations_for

    opts = opts or EngineOptions()
    opts.validate()
    if opts.algorithm not in _SSR_EVALUATORS:  # engine.py:246-250
        raise ValueError(f"algorithm {opts.algorithm!r} does not evaluate compiled automata")
    _check_vertex(g, source)
    t0 = time.monotonic()
    pq = partitioned_query(g, n, group)
    table = pq.table
    if table.starts.size and opts.timeout <= 0:  # _Clock.check(0), engine.py:87-89
        raise QueryTimeout(time.monotonic() - t0, 0)
    words, its, _ = pq.run(int(source), opts.timeout)
    return EvalResult(None, _iterations_for(opts.algorithm, its, table.starts.size), time.monotonic() - t0,
                      opts.algorithm, bits=words, nv=g.num_vertices)
