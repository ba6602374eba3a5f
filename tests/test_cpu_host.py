"""CPU-only tests: the C ABI library loads and exports its header, the host
logic mirrors the reference's (options, automaton reading, reverse, errors),
and the synthetic generators are deterministic."""

import ctypes
import glob
import math
import os
import re
import subprocess
import sys

import numpy as np
import pytest

from fixtures import automaton, host_graph, oracle_graph

import paper_2412_10287_b200 as P
from paper_2412_10287_b200 import _build, _lib, datagen
from paper_2412_10287_b200.automaton import reverse, transition_table

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    syms = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        syms |= set(re.findall(r"RPQ_API\s+[\w\s\*]+?\b(rpq_\w+)\s*\(", open(h).read()))
    return syms


def test_engine_library_exports_header():
    syms = _header_symbols()
    assert len(syms) >= 17
    lib = ctypes.CDLL(_build.ENGINE_SO)
    for s in syms:
        assert hasattr(lib, s), s
    # the ctypes binding covers exactly the header
    assert syms == set(_lib.ENGINE_SIGNATURES)
    assert _lib.engine().rpq_abi_version() == _lib.ABI_VERSION == 3


def test_header_constants_match_the_binding():
    """Status codes and tuning keys: include/rpq_b200.h and _lib.py agree."""
    text = open(os.path.join(ROOT, "include", "rpq_b200.h")).read()
    defs = dict((k, int(v)) for k, v in re.findall(r"#define (RPQ_\w+)\s+(\d+)\b", text))
    tune = {k[len("RPQ_TUNE_"):]: v for k, v in defs.items() if k.startswith("RPQ_TUNE_")}
    assert len(tune) >= 7
    for name, value in tune.items():
        assert getattr(_lib, "TUNE_" + name) == value, name
    for name in ("RPQ_OK", "RPQ_EINVAL", "RPQ_ERANGE", "RPQ_ETIMEOUT", "RPQ_ECUDA"):
        assert getattr(_lib, name) == defs[name], name
    assert _lib.BATCH == defs["RPQ_BATCH"] and _lib.STATS_LEVELS == defs["RPQ_STATS_LEVELS"]


def test_engine_library_is_sm100a_only():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _build.ENGINE_SO],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert all("sm_100a" in line for line in out.splitlines() if line.strip())


def test_c_abi_errors_without_device():
    lib = _lib.engine()
    h = ctypes.c_void_p()
    assert lib.rpq_graph_create(-1, 0, 0, ctypes.byref(h)) == _lib.RPQ_EINVAL
    assert lib.rpq_query_run(None, 0, 0.0, None) == _lib.RPQ_EINVAL
    assert lib.rpq_graph_destroy(None) == _lib.RPQ_OK
    assert "null" in _lib.last_error() or _lib.last_error() == ""


def test_options_validation():
    with pytest.raises(ValueError):
        P.EngineOptions(algorithm="quantum").validate()
    with pytest.raises(ValueError):
        P.EngineOptions(product_order="middle").validate()
    with pytest.raises(ValueError):
        P.EngineOptions(switch_threshold=-1).validate()
    g = P.LabeledGraph.from_edges(3, ["a"], [(0, 0, 1)])
    n = P.Automaton.build(1, {(0, False): [(0, 0)]}, [0], [0])
    with pytest.raises(ValueError):
        P.eval_ssr(g, n, 0, P.EngineOptions(algorithm="plan"))
    with pytest.raises(IndexError):
        P.eval_ssr(g, n, 3, P.EngineOptions())
    with pytest.raises(IndexError):
        P.eval_ssr(g, n, -1, P.EngineOptions())
    with pytest.raises(IndexError):
        P.eval_sdr(g, n, 7, P.EngineOptions())


def test_transition_table_follows_alphabet():
    # engine.py:99 iterates sorted(n.alphabet); labels >= num_labels are skipped
    n = P.Automaton.build(2, {(0, False): [(0, 1)], (1, True): [(1, 1)], (5, False): [(0, 0)]},
                          [0], [1])
    t = transition_table(n, num_labels=2)
    assert t.t_label.tolist() == [0, 1] and t.t_inv.tolist() == [0, 1]
    assert t.t_src.tolist() == [0, 1] and t.t_dst.tolist() == [1, 1]
    assert t.starts.tolist() == [0] and t.finals.tolist() == [1]
    # a symbol in the alphabet but not in transitions: KeyError, as in the reference
    bad = P.Automaton.build(1, {(0, False): [(0, 0)]}, [0], [0], alphabet=[(0, False), (1, False)])
    with pytest.raises(KeyError):
        transition_table(bad, num_labels=2)
    # transitions outside the alphabet are ignored
    sub = P.Automaton.build(1, {(0, False): [(0, 0)], (1, False): [(0, 0)]}, [0], [0],
                            alphabet=[(1, False)])
    assert transition_table(sub, 2).t_label.tolist() == [1]


def test_reverse_matches_reference_structure(reference_instances):
    # query_compiler.py:488-502: transposed matrices, flipped direction, swapped ends
    for rec in reference_instances[:200]:
        n = automaton(rec["nfa"])
        r = reverse(n)
        assert r.start_set == n.final_set and r.final_set == n.start_set
        for (idx, inv), m in n.transitions.items():
            rm = r.transitions[(idx, not inv)]
            assert sorted((b, a) for a, b in m.pairs()) == sorted(rm.pairs())
        assert r.alphabet == frozenset(r.transitions)
        assert reverse(r).transitions.keys() == n.transitions.keys()


def test_host_graph_mirrors_reference_layout(reference_instances):
    for rec in reference_instances[:100]:
        g = host_graph(rec["graph"])
        og = oracle_graph(rec["graph"])
        for l in range(g.num_labels):
            for inv in (False, True):
                m = g.adjacency(l, inv)
                indptr, indices = og.slot_csr(l, inv)
                assert np.array_equal(m.indptr, indptr)
                assert np.array_equal(m.indices, indices)


def test_generators_deterministic_and_canonical():
    a = datagen.generate("cfg1")
    b = datagen.generate("cfg1")
    assert a.digest() == b.digest()
    assert a.ne == 100_000 and a.nv == 10_000
    r = datagen.gen_rmat(12, 16, 8, 1.0, seed=7)
    assert not np.any(r.src == r.dst)  # self-loops dropped
    keys = r.src.astype(np.int64) << 32 | r.dst.astype(np.int64)
    assert np.all(np.diff(keys) > 0)  # sorted, (u, v) unique
    counts = np.bincount(r.lab, minlength=8)
    assert np.all(np.diff(counts) < 0)  # Zipf: rank frequencies decrease
    # label CSR built by the package equals the oracle's independent build
    g = r.labeled_graph()
    from oracle import OracleGraph

    og = OracleGraph(r.nv, r.nl, r.src, r.dst, r.lab)
    for l in (0, 3):
        for inv in (False, True):
            indptr, indices = og.slot_csr(l, inv)
            m = g.adjacency(l, inv)
            assert np.array_equal(m.indptr, indptr) and np.array_equal(m.indices, indices)


def test_generator_independent_of_thread_count():
    code = ("import sys; sys.path.insert(0, %r); from paper_2412_10287_b200 import datagen; "
            "print(datagen.gen_rmat(14, 16, 16, 1.0, seed=11).digest())" % ROOT)
    outs = set()
    for threads in ("1", "3"):
        env = dict(os.environ, OMP_NUM_THREADS=threads)
        outs.add(subprocess.run([sys.executable, "-c", code], env=env, capture_output=True,
                                text=True, check=True).stdout.strip())
    assert len(outs) == 1


def test_config_automata_are_the_reference_compilations():
    import json

    path = os.path.join(ROOT, "paper_2412_10287_b200", "data", "config_automata.json")
    d = json.load(open(path))
    # minimal DFA sizes of SURVEY.md Appendix B
    assert d["cfg1"]["a b*|min"]["nstates"] == 2
    assert d["cfg2"]["a ^b* c|min"]["nstates"] == 3
    assert d["cfg3"]["^a (b|c)* d|min"]["nstates"] == 3
    assert d["cfg5"][datagen.CHAIN16 + "|min"]["nstates"] == 9
    assert d["cfg5"][datagen.CHAIN16 + "|raw"]["nstates"] == 17
    for cfg in d.values():
        for nj in cfg.values():
            n = automaton(nj)
            assert n.nstates == nj["nstates"]
            assert math.isfinite(n.nstates)


def test_step_update_validates_shapes():
    from paper_2412_10287_b200.graph import CsrMatrix

    g = P.LabeledGraph.from_edges(3, ["a"], [(0, 0, 1)])
    n = P.Automaton.build(1, {(0, False): [(0, 0)]}, [0], [0])
    with pytest.raises(ValueError):  # test_engine.py:331-335
        P.step_update(CsrMatrix.from_pairs(1, 2, []), CsrMatrix.from_pairs(2, 1, []), g, n, P.EngineOptions())
    with pytest.raises(ValueError):
        P.step_update(CsrMatrix.from_pairs(2, 3, []), CsrMatrix.from_pairs(2, 3, []), g, n, P.EngineOptions())


def test_plan_ast_helpers():
    from paper_2412_10287_b200 import plan

    ast = plan.Concat((plan.Label("a"), plan.Star(plan.Label("b", True)), plan.Opt(plan.Label("c"))))
    r = plan.reverse_ast(ast)  # query_compiler.py:77-90
    assert r == plan.Concat((plan.Opt(plan.Label("c", True)), plan.Star(plan.Label("b", False)),
                             plan.Label("a", True)))
    assert plan.reverse_ast(r) == ast
    d = {"k": "alt", "c": [{"k": "label", "name": "a", "inv": False},
                           {"k": "plus", "c": {"k": "label", "name": "zz", "inv": True}}]}
    assert plan.ast_from_json(d) == plan.Alt((plan.Label("a"), plan.Plus(plan.Label("zz", True))))
    g = P.LabeledGraph.from_edges(3, ["a"], [(0, 0, 1)])
    with pytest.raises(ValueError):
        plan.eval_plan(g, plan.Label("a"), ("middle", 0), P.EngineOptions())
    with pytest.raises(IndexError):
        plan.eval_plan(g, plan.Label("a"), ("source", 3), P.EngineOptions())


def test_answer_set_view_matches_the_reference_set():
    """EvalResult.answer_set: the lazy set[int] a drop-in shim hands to the
    reference's EvalResult (engine.py:71-76) instead of building `reachable`."""
    import numpy as np

    from paper_2412_10287_b200.engine import EvalResult

    rng = np.random.default_rng(7)
    nv = 5000
    reach = (rng.random(nv) < 0.1).astype(np.uint8)
    want = set(np.flatnonzero(reach).tolist())
    bits = np.packbits(reach, bitorder="little")
    bits = np.concatenate([bits, np.zeros(-bits.size % 4, np.uint8)]).view(np.uint32)
    for kw in ({"bits": bits}, {"bits": bits, "count": len(want)}):
        r = EvalResult(None, 3, 0.0, "hybrid", nv=nv, **kw)
        a = r.answer_set
        assert len(a) == len(want) and a == want and want == a and set(a) == want
        assert all((v in a) == (v in want) for v in range(-3, nv + 3))
        assert "7" not in a and None not in a
    # sparse answers kept as (word, bits) pairs decode the same way
    words = np.flatnonzero(bits)
    pairs = np.stack([words.astype(np.uint32), bits[words]], axis=1).reshape(-1)
    r = EvalResult(None, 3, 0.0, "hybrid", nv=nv, pairs=pairs)
    assert r.answer_set == want and r.reachable == want and np.array_equal(r.reach, reach)


def test_wide_automata_are_routed_past_the_table_limits():
    """engine._is_wide mirrors rpq_query_create's limits (csrc/ssr_kernel.cuh
    kMaxStates / kMaxGroups / kMaxSlots): such automata go to rpq_ssr_wide
    instead of raising (the reference evaluates any automaton)."""
    import re

    from paper_2412_10287_b200 import _lib, engine
    from paper_2412_10287_b200.automaton import TransitionTable

    src = open(os.path.join(ROOT, "paper_2412_10287_b200", "csrc", "ssr_kernel.cuh")).read()
    for name, val in (("kMaxStates", _lib.MAX_STATES), ("kMaxGroups", _lib.MAX_GROUPS), ("kMaxSlots", _lib.MAX_SLOTS)):
        assert int(re.search(rf"constexpr int {name} = (\d+);", src).group(1)) == val

    def table(nstates, trans):
        s, l, i, d = (np.array(x) for x in zip(*trans)) if trans else ([], [], [], [])
        return TransitionTable(nstates, s, l, i, d, [0], [0])

    assert not engine._is_wide(table(3, [(0, 0, 0, 1), (1, 1, 1, 2)]))
    assert not engine._is_wide(table(256, [(q, 0, 0, (q + 1) % 256) for q in range(256)]))
    assert engine._is_wide(table(257, [(0, 0, 0, 1)]))
    # 129 symbols (label, inverted) on 2 states
    assert engine._is_wide(table(2, [(0, l // 2, l % 2, 1) for l in range(129)]))
    assert not engine._is_wide(table(2, [(0, l // 2, l % 2, 1) for l in range(128)]))
    # 257 (state, symbol) groups on 129 states x 2 symbols
    assert engine._is_wide(table(129, [(q, 0, i, q) for q in range(129) for i in (0, 1)][:257]))
    assert not engine._is_wide(table(129, [(q, 0, i, q) for q in range(129) for i in (0, 1)][:256]))
