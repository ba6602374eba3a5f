"""How answers reach the host (engine.py eval path, rpq_query_eval_list):
pinned pool buffers written by the kernel, sparse answers as (word, bits)
pairs, dense ones as the bitmap, the C bitmap call, and the on-demand uint8
vector -- every form bit-exact against the CPU oracle."""

import ctypes
import gc
import math

import numpy as np
import pytest

import paper_2412_10287_b200 as P
from paper_2412_10287_b200 import _lib
from paper_2412_10287_b200.engine import _ANSWERS, _table_for
from paper_2412_10287_b200.graph import CsrMatrix, device_graph

pytestmark = pytest.mark.gpu

NV = 300_000  # >= 4096 answer words: the pinned-buffer path


def graph():
    """Label a: a star 0 -> 1..200000 (dense answer) and a chain 250000 ->
    250001 -> ... -> 250009 (sparse); label b: one edge 299998 -> 299999."""
    star = [(0, v) for v in range(1, 200_001)]
    chain = [(250_000 + i, 250_001 + i) for i in range(9)]
    a = CsrMatrix.from_pairs(NV, NV, star + chain)
    b = CsrMatrix.from_pairs(NV, NV, [(299_998, 299_999)])
    return P.LabeledGraph(NV, ["a", "b"], [a, b])


A_PLUS = P.Automaton.build(2, {(0, False): [(0, 1), (1, 1)]}, [0], [1])  # a+


def reach_of(src, g):
    # a+ from src: every vertex reachable by >= 1 a-edge (BFS on host, tiny)
    fwd = g.forward[0]
    seen, front = set(), {src}
    while front:
        nxt = set()
        for u in front:
            for v in fwd.indices[fwd.indptr[u]:fwd.indptr[u + 1]]:
                if v not in seen:
                    seen.add(int(v))
                    nxt.add(int(v))
        front = nxt
    out = np.zeros(NV, dtype=np.uint8)
    out[list(seen)] = 1
    return out


@pytest.mark.parametrize("source,kind", [(0, "dense"), (250_000, "sparse"), (123, "empty"), (299_998, "empty")])
def test_eval_answer_forms(source, kind):
    g = graph()
    want = reach_of(source, g)
    for kernel in ("auto", "grid"):
        r = P.eval_ssr(g, A_PLUS, source, P.EngineOptions(timeout=math.inf, kernel=kernel))
        assert np.array_equal(r.reach, want), (source, kernel)
        assert r.bits.size == (NV + 31) // 32
        assert len(r.reachable) == int(want.sum())


def test_list_and_bitmap_calls_agree():
    g = graph()
    dg = device_graph(g)
    table = _table_for(A_PLUS, g.num_labels)
    dg.ensure_labels(table.labels)
    q = dg.acquire_query(table)
    lib = _lib.engine()
    nwords = (NV + 31) // 32
    try:
        for source in (0, 250_000, 7):
            want = reach_of(source, g)
            st = _lib.RpqStats()
            buf = _ANSWERS.take(nwords)
            assert lib.rpq_query_eval_list(q, source, -1.0, 0, 0, 4.0, 0, ctypes.byref(st), buf.ctypes.data,
                                           nwords) == 0, _lib.last_error()
            packed = np.zeros(nwords * 4, dtype=np.uint8)
            packed[: (NV + 7) // 8] = np.packbits(want, bitorder="little")
            nz = int(np.count_nonzero(packed.view(np.uint32)))
            if 2 * nz < nwords:
                assert st.answer_list == 1 and st.answer_words == nz
                pairs = buf[: 2 * nz]
                bits = np.zeros(nwords, dtype=np.uint32)
                bits[pairs[0::2]] = pairs[1::2]
            else:
                assert st.answer_list == 0
                bits = buf.copy()
            got = np.unpackbits(bits.view(np.uint8), bitorder="little")[:NV]
            assert np.array_equal(got, want), source
            # the plain C call always returns the bitmap, pinned or not
            for out in (np.zeros(nwords, dtype=np.uint32), _ANSWERS.take(nwords)):
                assert lib.rpq_query_eval(q, source, -1.0, 0, 0, 4.0, 0, ctypes.byref(st), out.ctypes.data,
                                          nwords) == 0
                got = np.unpackbits(out.view(np.uint8), bitorder="little")[:NV]
                assert np.array_equal(got, want), source
            # the uint8 vector, expanded on demand from the last run's bitmap
            r8 = np.zeros(NV, dtype=np.uint8)
            assert lib.rpq_query_copy_reach(q, _lib.ptr(r8, ctypes.c_uint8)) == 0
            assert np.array_equal(r8, want)
    finally:
        dg.release_query(table, q)


def test_pool_buffers_are_recycled():
    g = graph()
    opts = P.EngineOptions(timeout=math.inf, kernel="grid")
    results = [P.eval_ssr(g, A_PLUS, 0, opts) for _ in range(3)]
    ptrs = {r.bits.ctypes.data for r in results}
    assert len(ptrs) == 3  # live results never share a buffer
    del results
    gc.collect()
    again = P.eval_ssr(g, A_PLUS, 0, opts)
    assert again.bits.ctypes.data in ptrs  # a freed buffer came back from the pool
    assert np.array_equal(again.reach, reach_of(0, g))
