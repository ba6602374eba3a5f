"""Drop-in query API: the reference engine's names, arguments and errors
(/root/reference/pkg/src/rpq/engine.py), evaluated by the sm_100a kernel.

    eval_ssr(g, n, source, opts) -> EvalResult          engine.py:242-251
    eval_ssr_masked / eval_ssr_no_mask / eval_ssr_hybrid engine.py:146-232
    eval_sdr(g, n, target, opts, algorithm=None)        engine.py:254-266
    step_update(m, p, g, n, opts)                       engine.py:127-138
    EngineOptions, EvalResult, QueryTimeout             engine.py:45-89

``g`` is the reference's LabeledGraph (or this package's host mirror), ``n``
its compiled TwoNfa.  The three SSR algorithms of the reference compute the
same P, level by level (Alg. 1 and Alg. 2 of PAPER.md differ only in how
much of P they re-expand), so all three run the same device BFS; the
``algorithm`` tag is kept in the result and the iteration count follows each
loop's own accounting.  There is no CPU path: the CUDA library must load.
"""

import collections.abc
import ctypes
import dataclasses
import math
import threading
import time
import weakref
from dataclasses import dataclass

import numpy as np

from . import _lib
from .automaton import reverse, transition_table
from .graph import device_graph

ALGORITHMS = ("masked", "no_mask", "hybrid", "plan")
DIRECTIONS = {"auto": _lib.DIR_AUTO, "push": _lib.DIR_PUSH, "pull": _lib.DIR_PULL}


class QueryTimeout(RuntimeError):
    """Evaluation exceeded the wall-clock budget (engine.py:45-51)."""

    def __init__(self, elapsed: float, iterations: int):
        super().__init__(f"query timed out after {elapsed:.3f}s ({iterations} iterations)")
        self.elapsed = elapsed
        self.iterations = iterations


class EngineError(RuntimeError):
    """A CUDA or internal failure of the device engine."""


@dataclass
class EngineOptions:
    """engine.py:54-68, plus ``device`` (CUDA ordinal the graph lives on)."""

    algorithm: str = "hybrid"
    switch_threshold: float = 100
    product_order: str = "left"
    timeout: float = 60.0
    debug_checks: bool = False
    device: int = 0
    direction: str = "auto"  # per-level push/pull policy of the device BFS
    alpha: float = 4.0  # Beamer's switch constant (pull when m_f * alpha > m_u)
    count_te: bool = False  # exact product-edge count in EvalResult.stats
    kernel: str = "auto"  # "auto": small state spaces run on one CTA; "grid": always the grid kernel

    def validate(self) -> None:
        if self.kernel not in ("auto", "grid"):
            raise ValueError(f"unknown kernel {self.kernel!r}")
        if self.direction not in DIRECTIONS:
            raise ValueError(f"unknown direction {self.direction!r}")
        if not self.alpha > 0:
            raise ValueError("alpha must be > 0")
        if self.algorithm not in ALGORITHMS:
            raise ValueError(f"unknown algorithm {self.algorithm!r}")
        if self.product_order not in ("left", "right"):
            raise ValueError(f"unknown product order {self.product_order!r}")
        if self.switch_threshold < 0:
            raise ValueError("switch threshold must be >= 0")


class AnswerSet(collections.abc.Set):
    """A read-only ``set[int]`` view of an answer as the device returned it
    (bitmap or sparse pairs): membership is one bit test, ``len`` the device's
    answer count, iteration decodes on demand.  Compares equal to the
    reference's ``set`` of the same vertices.  For callers that would
    otherwise build the reference's ``reachable`` set (about 0.05 us per
    answer vertex in CPython: 120 ms for cfg3's 2.3M answers)."""

    __slots__ = ("_res",)

    def __init__(self, res):
        self._res = res

    def __contains__(self, v):
        try:
            v = int(v)
        except (TypeError, ValueError):
            return False
        res = self._res
        if not 0 <= v < res._nv:
            return False
        if res._reachable is not None:
            return v in res._reachable
        return bool((int(res.bits[v >> 5]) >> (v & 31)) & 1)

    def __len__(self):
        return self._res.count

    def __iter__(self):
        return iter(np.flatnonzero(self._res.reach).tolist())

    def __repr__(self):
        return f"AnswerSet(|V|={self._res._nv}, size={len(self)})"

    __hash__ = None


class EvalResult:
    """Result of one evaluation (engine.py:71-76).

    ``reachable`` is the reference's ``set[int]`` of answer vertices, built on
    first access from ``reach``, the device's ``uint8[|V|]`` answer vector.
    """

    __slots__ = ("_reach", "_bits", "_pairs", "_nv", "_reachable", "_count", "iterations", "elapsed", "algorithm",
                 "stats")

    def __init__(self, reach, iterations, elapsed, algorithm, stats=None, bits=None, nv=None, pairs=None,
                 count=None):
        self._count = count  # |answer| as counted on the device, if known
        self._reach = reach
        self._bits = bits  # answer bitmap as read back from the device (uint32 words)
        self._pairs = pairs  # or a sparse answer as read back: (word index, word) uint32 pairs
        self._nv = nv
        self._reachable = None
        self.iterations = iterations
        self.elapsed = elapsed
        self.algorithm = algorithm
        self.stats = stats

    @property
    def reach(self):
        """uint8[|V|]: 1 where the vertex is an answer (decoded on first use)."""
        if self._reach is None:
            self._reach = bits_to_reach(self.bits, self._nv)
        return self._reach

    @property
    def bits(self):
        """The answer as uint32 words, bit v % 32 of word v // 32."""
        if self._bits is None and self._pairs is not None:
            bits = np.zeros((self._nv + 31) // 32, dtype=np.uint32)
            bits[self._pairs[0::2]] = self._pairs[1::2]
            self._bits, self._pairs = bits, None
        if self._bits is None:
            packed = np.packbits(self._reach, bitorder="little")
            packed = np.concatenate([packed, np.zeros(-packed.size % 4, dtype=np.uint8)])
            self._bits = packed.view(np.uint32)
        return self._bits

    @property
    def count(self):
        """|answer| (the device's count when it came with the result)."""
        if self._count is None:
            if self._reachable is not None:
                self._count = len(self._reachable)
            else:
                self._count = int(np.bitwise_count(self.bits).sum()) if self._nv else 0
        return self._count

    @property
    def answer_set(self):
        """The answer as a lazy read-only set (AnswerSet): what a drop-in shim
        hands to the reference's EvalResult instead of building ``reachable``."""
        return AnswerSet(self)

    @property
    def reachable(self):
        if self._reachable is None:
            self._reachable = set(np.flatnonzero(self.reach).tolist())
        return self._reachable

    def __eq__(self, other):
        if not isinstance(other, EvalResult):
            return NotImplemented
        return (self.reachable == other.reachable and self.iterations == other.iterations
                and self.algorithm == other.algorithm)

    __hash__ = None

    def __repr__(self):
        return (f"EvalResult(|reachable|={len(self.reachable)}, "
                f"iterations={self.iterations}, elapsed={self.elapsed:.6f}, "
                f"algorithm={self.algorithm!r})")


def raise_for_status(rc, what=""):
    """Map a C-ABI status to the reference's exception types."""
    if rc == _lib.RPQ_OK:
        return
    msg = _lib.last_error()
    text = f"{what}: {msg}" if what else msg
    if rc == _lib.RPQ_EINVAL:
        raise ValueError(text)
    if rc == _lib.RPQ_ERANGE:
        raise IndexError(text)
    if rc == _lib.RPQ_ENOMEM:
        raise MemoryError(text)
    if rc == _lib.RPQ_ENOLABEL:
        raise ValueError(text)
    raise EngineError(text)


def _check_vertex(g, vertex):
    """engine.py:141-143"""
    if not 0 <= vertex < g.num_vertices:
        raise IndexError(f"vertex index {vertex} out of range")


def _iterations_for(algorithm, masked_iterations, nstarts):
    # The masked loop runs `while m.nnz` and so does zero iterations when the
    # automaton has no start state; the mask-free and hybrid loops always run
    # at least one (engine.py:157, :184, :209).  Otherwise all three count
    # the D+1 steps of a BFS of depth D.
    if nstarts == 0 and algorithm in ("no_mask", "hybrid"):
        return 1
    return masked_iterations


_TABLES = {}  # id(automaton) -> (weakref, num_labels, TransitionTable)


def _table_for(n, num_labels):
    """transition_table(n, num_labels), cached per automaton object (compiled
    automata are not mutated after compile; query_compiler.py treats them as
    values)."""
    hit = _TABLES.get(id(n))
    if hit is not None and hit[0]() is n and hit[1] == num_labels:
        return hit[2]
    table = transition_table(n, num_labels)
    try:
        ref = weakref.ref(n, lambda _r, k=id(n): _TABLES.pop(k, None))
    except TypeError:
        return table
    _TABLES[id(n)] = (ref, num_labels, table)
    return table


def bits_to_reach(words, nv):
    """uint8[nv] answer vector from the answer bitmap (bit v%32 of word v/32)."""
    return np.unpackbits(words.view(np.uint8), bitorder="little")[:nv]


class _AnswerPool:
    """Pinned, device-mapped host bitmaps for eval_ssr answers (rpq_host_alloc).
    The kernel's epilogue writes the answer straight into one over PCIe, and
    the EvalResult keeps it as its ``bits`` array: no copy node, no host
    memcpy, no page faults on a fresh array.  A buffer returns to the pool when
    the last array viewing it is garbage-collected."""

    KEEP = 16  # free buffers kept per size

    def __init__(self):
        self._free = {}
        self._lock = threading.Lock()

    def take(self, nwords):
        with self._lock:
            lst = self._free.get(nwords)
            ptr = lst.pop() if lst else None
        if ptr is None:
            p = ctypes.c_void_p()
            raise_for_status(_lib.engine().rpq_host_alloc(nwords * 4, ctypes.byref(p)), "rpq_host_alloc")
            ptr = p.value
        buf = (ctypes.c_uint32 * nwords).from_address(ptr)
        weakref.finalize(buf, self._give, nwords, ptr)
        return np.ctypeslib.as_array(buf)

    def _give(self, nwords, ptr):
        with self._lock:
            lst = self._free.setdefault(nwords, [])
            if len(lst) < self.KEEP:
                lst.append(ptr)
                return
        try:
            _lib.engine().rpq_host_free(ptr)
        except Exception:  # interpreter shutdown
            pass


_ANSWERS = _AnswerPool()

_TLS = threading.local()


def _thread_stats():
    """One rpq_stats block per thread, reused by every eval_ssr call."""
    st = getattr(_TLS, "stats", None)
    if st is None:
        st = _TLS.stats = _lib.RpqStats()
    return st


def _is_wide(table):
    """True when the automaton exceeds the persistent kernel's table limits
    (more than 256 states or (state, symbol) groups, more than 128 symbols).
    The reference has no such limit (engine.py:99-102 iterates N.alphabet)."""
    if table.nstates > _lib.MAX_STATES:
        return True
    if table.t_src.size <= _lib.MAX_SLOTS:
        return False
    sym = table.t_label.astype(np.int64) * 2 + table.t_inv
    if np.unique(sym).size > _lib.MAX_SLOTS:
        return True
    return np.unique(table.t_src.astype(np.int64) * (2 << 32) + sym).size > _lib.MAX_GROUPS


def _run_wide(g, dg, table, source, opts, tag, t0, want_stats):
    """eval_ssr for automata beyond the kernel tables: rpq_ssr_wide, one device
    push step per level over the transition list (same answer, same counts)."""
    lib = _lib.engine()
    remaining = opts.timeout - (time.monotonic() - t0)
    first_check = not (tag == "masked" and table.starts.size == 0)
    if first_check and (remaining < 0 or opts.timeout <= 0):
        raise QueryTimeout(time.monotonic() - t0, 0)
    budget = -1.0 if math.isinf(remaining) else max(remaining, 0.0)
    nwords = (g.num_vertices + 31) // 32
    words = np.zeros(max(nwords, 1), dtype=np.uint32)
    stats = _lib.RpqStats()
    rc = lib.rpq_ssr_wide(dg.handle, table.nstates, table.t_src.size, _lib.ptr(table.t_src, ctypes.c_int32),
                          _lib.ptr(table.t_label, ctypes.c_int32), _lib.ptr(table.t_inv, ctypes.c_uint8),
                          _lib.ptr(table.t_dst, ctypes.c_int32), table.starts.size,
                          _lib.ptr(table.starts, ctypes.c_int32), table.finals.size,
                          _lib.ptr(table.finals, ctypes.c_int32), int(source), budget,
                          _lib.ptr(words, ctypes.c_uint32), words.size, ctypes.byref(stats))
    if rc == _lib.RPQ_ETIMEOUT:
        raise QueryTimeout(time.monotonic() - t0, _iterations_for(tag, stats.iterations, table.starts.size))
    raise_for_status(rc, "rpq_ssr_wide")
    iterations = _iterations_for(tag, stats.iterations, table.starts.size)
    return EvalResult(None, iterations, time.monotonic() - t0, tag,
                      stats.to_dict() if want_stats or opts.debug_checks or opts.count_te else None,
                      bits=words[:nwords], nv=g.num_vertices, pairs=None, count=int(stats.reach_count))


def _run(g, n, source, opts, tag, *, want_stats=False):
    opts.validate()
    _check_vertex(g, source)
    t0 = time.monotonic()
    dg = device_graph(g, opts.device)
    table = _table_for(n, g.num_labels)
    dg.ensure_labels(table.labels)
    if _is_wide(table):
        return _run_wide(g, dg, table, source, opts, tag, t0, want_stats)
    lib = _lib.engine()
    q = dg.acquire_query(table)
    try:
        # _Clock.check(0) at the top of the first iteration (engine.py:87-89).
        # The masked loop (`while m.nnz`, engine.py:157) never reaches it when
        # the automaton has no start state, so that case returns normally.
        remaining = opts.timeout - (time.monotonic() - t0)
        first_check = not (tag == "masked" and table.starts.size == 0)
        if first_check and (remaining < 0 or opts.timeout <= 0):
            raise QueryTimeout(time.monotonic() - t0, 0)
        budget = -1.0 if math.isinf(remaining) else max(remaining, 0.0)
        nwords = (g.num_vertices + 31) // 32
        # large answers land in a pinned buffer the kernel writes directly
        words = _ANSWERS.take(nwords) if nwords >= 4096 else np.empty(nwords, dtype=np.uint32)
        stats = _thread_stats()  # read (or copied out) before this thread's next call
        # options, run, wait and the answer bitmap in one C call (raw addresses)
        rc = lib.rpq_query_eval_list(q, int(source), budget, DIRECTIONS[opts.direction],
                                     int(opts.count_te or opts.debug_checks), opts.alpha,
                                     1 if opts.kernel == "auto" else 0, ctypes.addressof(stats),
                                     words.ctypes.data if words.size else None, words.size)
        if rc == _lib.RPQ_ETIMEOUT:
            raise QueryTimeout(time.monotonic() - t0,
                               _iterations_for(tag, stats.iterations, table.starts.size))
        raise_for_status(rc, "rpq_query_eval")
        iterations = _iterations_for(tag, stats.iterations, table.starts.size)
        pairs = None
        if stats.answer_list:
            # a sparse answer came back as (word index, word) pairs: keep a
            # copy of them (the bitmap is built on first use) and let the
            # pinned buffer go back to the pool
            pairs = words[: 2 * int(stats.answer_words)].copy()
            words = None
        if opts.debug_checks:
            _debug_invariants(lib, q, table, g.num_vertices, stats, iterations)
    finally:
        dg.release_query(table, q)
    return EvalResult(None, iterations, time.monotonic() - t0, tag,
                      stats.to_dict() if want_stats or opts.debug_checks or opts.count_te else None,
                      bits=words, nv=g.num_vertices, pairs=pairs, count=int(stats.reach_count))


def _debug_invariants(lib, q, table, nv, stats, iterations):
    """Executable invariants of debug mode (engine.py:161-170, :187-190):
    P grew by exactly the disjoint per-level frontiers, and the loop stayed
    within |Q|*|V| iterations."""
    words = (nv + 31) // 32
    buf = np.zeros(max(words * table.nstates, 1), dtype=np.uint32)
    raise_for_status(lib.rpq_query_copy_visited(q, _lib.ptr(buf, ctypes.c_uint32), buf.size),
                     "rpq_query_copy_visited")
    popcount = int(np.unpackbits(buf.view(np.uint8)).sum())
    levels = stats.level_new[:min(stats.iterations + 1, _lib.STATS_LEVELS)]
    assert popcount == stats.visited_pairs, "visited set is not the union of the frontiers"
    if stats.iterations < _lib.STATS_LEVELS:
        assert sum(levels) == stats.visited_pairs, "frontiers overlap or were lost"
    assert iterations <= table.nstates * nv or nv == 0, "exceeded |Q|*|V| iterations"
    reach = int(stats.reach_count)
    assert 0 <= reach <= nv


def eval_ssr_masked(g, n, source, opts):
    """Frontier/visited iteration (Alg. 1; engine.py:146-171)."""
    return _run(g, n, source, opts, "masked")


def eval_ssr_no_mask(g, n, source, opts):
    """Single-accumulator iteration (Alg. 2; engine.py:174-194)."""
    return _run(g, n, source, opts, "no_mask")


def eval_ssr_hybrid(g, n, source, opts):
    """Mask-free until nnz(P) > switch_threshold, masked after (engine.py:197-232)."""
    return _run(g, n, source, opts, "hybrid")


_SSR_EVALUATORS = {
    "masked": eval_ssr_masked,
    "no_mask": eval_ssr_no_mask,
    "hybrid": eval_ssr_hybrid,
}


def eval_ssr(g, n, source, opts):
    """Dispatch on ``opts.algorithm`` (engine.py:242-251)."""
    opts.validate()
    try:
        evaluator = _SSR_EVALUATORS[opts.algorithm]
    except KeyError:
        raise ValueError(
            f"algorithm {opts.algorithm!r} does not evaluate compiled automata"
        ) from None
    return evaluator(g, n, source, opts)


def eval_sdr(g, n, target, opts, algorithm=None):
    """Single-destination reachability: SSR from the target over the reversed
    automaton (engine.py:254-266)."""
    _check_vertex(g, target)
    if algorithm is not None:
        opts = dataclasses.replace(opts, algorithm=algorithm)
    return eval_ssr(g, reverse(n), target, opts)


def eval_ssr_batch(g, n, sources, opts, *, stats=None):
    """uint8[len(sources), |V|]: row i is eval_ssr(g, n, sources[i], opts)'s answer.

    Defined as the per-source loop; the reference has no
    multi-source entry point.  Evaluated 64 sources per kernel launch with
    bit-sliced frontiers (batch_kernel.cuh).  ``opts.timeout`` bounds each
    launch of up to 64 sources.  If ``stats`` is a list, the statistics of
    every launch are appended to it."""
    opts.validate()
    sources = [int(s) for s in sources]
    for s in sources:
        _check_vertex(g, s)
    nv = int(g.num_vertices)
    out = np.zeros((len(sources), nv), dtype=np.uint8)
    if not sources:
        return out
    t0 = time.monotonic()
    dg = device_graph(g, opts.device)
    table = _table_for(n, g.num_labels)
    dg.ensure_labels(table.labels)
    lib = _lib.engine()
    q = dg.acquire_query(table)
    try:
        words = (nv + 31) // 32
        bits = np.zeros((_lib.BATCH, max(words, 1)), dtype=np.uint32)
        for b0 in range(0, len(sources), _lib.BATCH):
            chunk = np.ascontiguousarray(sources[b0:b0 + _lib.BATCH], dtype=np.int32)
            # _Clock.check(0), engine.py:87-89: a zero or negative budget has
            # already expired (the C side reads a negative budget as "none")
            if opts.timeout <= 0 and table.starts.size:
                raise QueryTimeout(time.monotonic() - t0, 0)
            budget = -1.0 if math.isinf(opts.timeout) else max(float(opts.timeout), 0.0)
            raise_for_status(lib.rpq_query_run_batch(q, chunk.size, _lib.ptr(chunk, ctypes.c_int32), budget,
                                                     None), "rpq_query_run_batch")
            st = _lib.RpqBatchStats()
            rc = lib.rpq_query_wait_batch(q, ctypes.byref(st))
            if rc == _lib.RPQ_ETIMEOUT:
                raise QueryTimeout(time.monotonic() - t0, int(st.levels))
            raise_for_status(rc, "rpq_query_wait_batch")
            if stats is not None:
                stats.append(st.to_dict())
            if nv:
                raise_for_status(lib.rpq_query_copy_batch_bits(q, _lib.ptr(bits, ctypes.c_uint32), bits.shape[1]),
                                 "rpq_query_copy_batch_bits")
                rows = np.unpackbits(bits[: chunk.size].view(np.uint8), axis=1, bitorder="little")
                out[b0:b0 + chunk.size] = rows[:, :nv]
    finally:
        dg.release_query(table, q)
    return out


def _csr_to_bits(m, nstates, nv):
    words = (nv + 31) // 32
    out = np.zeros((nstates, max(words, 1)), dtype=np.uint32)
    indptr = np.asarray(m.indptr, dtype=np.int64)
    cols = np.asarray(m.indices, dtype=np.int64)
    rows = np.repeat(np.arange(indptr.size - 1, dtype=np.int64), np.diff(indptr))
    if cols.size:
        np.bitwise_or.at(out, (rows, cols >> 5), (np.uint32(1) << (cols & 31).astype(np.uint32)))
    return out


def _bits_to_csr(bits, nv):
    nstates = bits.shape[0]
    dense = np.unpackbits(bits.view(np.uint8), axis=1, bitorder="little")[:, :nv]
    rows, cols = np.nonzero(dense)
    indptr = np.zeros(nstates + 1, dtype=np.int64)
    np.add.at(indptr, rows + 1, 1)
    np.cumsum(indptr, out=indptr)
    return indptr, cols.astype(np.int64)


def step_update(m, p, g, n, opts):
    """One traversal step (engine.py:127-138): the per-symbol products of the
    frontier ``m``, minus everything in ``p`` -- on the device.  ``m`` and
    ``p`` are |Q| x |V| Boolean matrices (the reference's SparseBoolMatrix or
    any object with nrows/ncols/indptr/indices); the result has m's type."""
    if m.shape != p.shape:
        raise ValueError(f"step_update: frontier {m.shape} vs visited {p.shape}")
    opts.validate()
    nstates, nv = m.shape
    if nstates != n.nstates or nv != g.num_vertices:
        raise ValueError(f"step_update: matrices must be {n.nstates}x{g.num_vertices}, got {m.shape}")
    dg = device_graph(g, opts.device)
    table = _table_for(n, g.num_labels)
    dg.ensure_labels(table.labels)
    lib = _lib.engine()
    q = dg.acquire_query(table)
    try:
        mb = _csr_to_bits(m, nstates, nv)
        pb = _csr_to_bits(p, nstates, nv)
        out = np.zeros_like(mb)
        if nv:
            raise_for_status(lib.rpq_query_step(q, _lib.ptr(mb, ctypes.c_uint32), _lib.ptr(pb, ctypes.c_uint32),
                                                mb.shape[1], _lib.ptr(out, ctypes.c_uint32)), "rpq_query_step")
    finally:
        dg.release_query(table, q)
    indptr, indices = _bits_to_csr(out, nv)
    return type(m)(nstates, nv, indptr, indices)


class PreparedQuery:
    """An automaton bound to a device-resident graph, for callers that
    evaluate it many times (batches of sources, the bench).  ``launch`` only
    enqueues work on ``stream`` (a raw cudaStream_t handle, e.g.
    ``torch.cuda.current_stream().cuda_stream``); ``wait`` returns the run's
    statistics; ``reach`` copies the answer to the host."""

    def __init__(self, g, n, device=0):
        self.g = g
        self.dg = device_graph(g, device)
        self.table = transition_table(n, g.num_labels)
        self.dg.ensure_labels(self.table.labels)
        # a private handle: set_options / set_tuning change it for good
        self.q = self.dg.acquire_query(self.table, private=True)
        self.nv = int(g.num_vertices)

    def set_options(self, direction="auto", count_te=False, alpha=4.0):
        raise_for_status(_lib.engine().rpq_query_set_options(
            self.q, DIRECTIONS[direction], int(count_te), float(alpha)), "rpq_query_set_options")

    def set_tuning(self, emit_mode=None, emit_inline_max=None, kernel=None):
        lib = _lib.engine()
        if kernel is not None:
            raise_for_status(lib.rpq_query_set_tuning(self.q, _lib.TUNE_SMALL, 1.0 if kernel == "auto" else 0.0),
                             "rpq_query_set_tuning")
        if emit_mode is not None:
            raise_for_status(lib.rpq_query_set_tuning(self.q, _lib.TUNE_EMIT_MODE, float(emit_mode)), "rpq_query_set_tuning")
        if emit_inline_max is not None:
            raise_for_status(lib.rpq_query_set_tuning(self.q, _lib.TUNE_EMIT_INLINE_MAX, float(emit_inline_max)),
                             "rpq_query_set_tuning")

    def launch(self, source, timeout=-1.0, stream=None):
        _check_vertex(self.g, source)
        raise_for_status(_lib.engine().rpq_query_run(self.q, int(source), float(timeout), stream),
                         "rpq_query_run")

    def wait(self):
        stats = _lib.RpqStats()
        rc = _lib.engine().rpq_query_wait(self.q, ctypes.byref(stats))
        if rc == _lib.RPQ_ETIMEOUT:
            raise QueryTimeout(stats.device_ms / 1e3, stats.iterations)
        raise_for_status(rc, "rpq_query_wait")
        return stats

    def launch_batch(self, sources, timeout=-1.0, stream=None):
        """Enqueue one multi-source run (<= 64 sources, bit-sliced)."""
        src = np.ascontiguousarray([int(s) for s in sources], dtype=np.int32)
        for s in src:
            _check_vertex(self.g, int(s))
        self._batch_src = src  # keep alive until the copy is enqueued (synchronous here)
        raise_for_status(_lib.engine().rpq_query_run_batch(self.q, src.size, _lib.ptr(src, ctypes.c_int32),
                                                           float(timeout), stream), "rpq_query_run_batch")

    def wait_batch(self):
        stats = _lib.RpqBatchStats()
        rc = _lib.engine().rpq_query_wait_batch(self.q, ctypes.byref(stats))
        if rc == _lib.RPQ_ETIMEOUT:
            raise QueryTimeout(stats.device_ms / 1e3, stats.levels)
        raise_for_status(rc, "rpq_query_wait_batch")
        return stats

    def batch_reach(self, nsrc):
        """uint8[nsrc, |V|] answers of the last batch run."""
        words = (self.nv + 31) // 32
        bits = np.zeros((nsrc, max(words, 1)), dtype=np.uint32)
        if self.nv:
            raise_for_status(_lib.engine().rpq_query_copy_batch_bits(self.q, _lib.ptr(bits, ctypes.c_uint32),
                                                                     bits.shape[1]), "rpq_query_copy_batch_bits")
        return np.unpackbits(bits.view(np.uint8), axis=1, bitorder="little")[:, : self.nv]

    def reach(self, out=None):
        out = np.empty(self.nv, dtype=np.uint8) if out is None else out
        if self.nv:
            raise_for_status(_lib.engine().rpq_query_copy_reach(self.q, _lib.ptr(out, ctypes.c_uint8)),
                             "rpq_query_copy_reach")
        return out

    def visited_counts(self):
        """Pairs of P per automaton state (popcount of each visited row)."""
        words = (self.nv + 31) // 32
        buf = np.zeros(max(words * self.table.nstates, 1), dtype=np.uint32)
        raise_for_status(_lib.engine().rpq_query_copy_visited(
            self.q, _lib.ptr(buf, ctypes.c_uint32), buf.size), "rpq_query_copy_visited")
        rows = buf[: words * self.table.nstates].reshape(self.table.nstates, words)
        return np.unpackbits(rows.view(np.uint8), axis=1).sum(axis=1).astype(np.int64)

    def io_bytes(self):
        h2d, d2h = ctypes.c_int64(), ctypes.c_int64()
        raise_for_status(_lib.engine().rpq_query_io_bytes(self.q, ctypes.byref(h2d), ctypes.byref(d2h)),
                         "rpq_query_io_bytes")
        return int(h2d.value), int(d2h.value)

    def close(self):
        if self.q is not None:
            self.dg.destroy_query(self.q)
            self.q = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
