"""Generate golden vectors by running the REFERENCE package itself.

Run in the build container only (it imports /root/reference, which does not
exist on the GPU box); the outputs are committed under tests/golden/ and
paper_2412_10287_b200/data/, and the tests read only those files.

    python tests/golden/make_golden.py random      # reference test-suite instances
    python tests/golden/make_golden.py automata    # compiled config queries
    python tests/golden/make_golden.py config cfg1 cfg2 [cfg3 cfg5 ...]
    python tests/golden/make_golden.py plan        # eval_plan (engine.py:292-390) on the same streams
    python tests/golden/make_golden.py desk        # test_acceptance.py criteria 7/8: desk-scale bench

Instance sources (each replays the reference test's own RNG stream):
  engine_random_15   test_engine.py:403-415 (seed 15, 40 instances, unknown label "zz")
  acceptance_c1      test_acceptance.py:60-84 (seed 0xC1, 500 instances)
  acceptance_c2      test_acceptance.py:92-112 (seed 0xC2, SSR/SDR duality, 100 instances)
  acceptance_c4      test_acceptance.py:141-153 (seed 0xC4, a* contains its source)
  hybrid_9           test_engine.py:269-279 (seed 9, switch thresholds 0/3/inf)
  known_answers      test_engine.py:103-171, :367-373 and test_oracle.py hand cases
"""

import base64
import gzip
import json
import math
import os
import random
import sys
import time

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REF_SRC)
sys.path.insert(0, REF_TESTS)
sys.path.insert(0, ROOT)

import helpers  # noqa: E402  (reference test helpers)
from rpq.engine import (  # noqa: E402
    EngineOptions,
    eval_plan,
    step_update,
    eval_sdr,
    eval_ssr,
    eval_ssr_hybrid,
    eval_ssr_masked,
    eval_ssr_no_mask,
)
from rpq.graph_store import LabeledGraph as RefGraph  # noqa: E402
from rpq.oracle import oracle_ssr  # noqa: E402
from rpq.query_compiler import compile as ref_compile  # noqa: E402
from rpq.query_compiler import parse_query  # noqa: E402
from rpq.sparse_bool import SparseBoolMatrix  # noqa: E402


def graph_json(g):
    return {
        "nv": g.num_vertices,
        "labels": list(g.labels),
        "vertices": list(g.vertices),
        "edges": [g.forward[l].pairs() for l in range(g.num_labels)],
    }


def nfa_json(n):
    return {
        "nstates": n.nstates,
        "transitions": [[k[0], bool(k[1]), [list(p) for p in m.pairs()]]
                        for k, m in sorted(n.transitions.items())],
        "alphabet": sorted([[a[0], bool(a[1])] for a in n.alphabet]),
        "starts": sorted(n.start_set),
        "finals": sorted(n.final_set),
        "label_names": {str(k): v for k, v in n.label_names.items()},
    }


def run_all(g, n, source, opts=None):
    opts = opts or EngineOptions(timeout=math.inf)
    m = eval_ssr_masked(g, n, source, opts)
    nm = eval_ssr_no_mask(g, n, source, opts)
    h = eval_ssr_hybrid(g, n, source, opts)
    assert m.reachable == nm.reachable == h.reachable
    return {
        "expected": sorted(h.reachable),
        "iterations": {"masked": m.iterations, "no_mask": nm.iterations,
                       "hybrid": h.iterations},
        "oracle_ssr": sorted(oracle_ssr(g, n, source)),
    }


def instance(g, n, source, tag, **extra):
    d = {"tag": tag, "graph": graph_json(g), "nfa": nfa_json(n), "source": source}
    d.update(run_all(g, n, source))
    d.update(extra)
    return d


def gen_random():
    out = []
    # test_engine.py:403-415
    rng = random.Random(15)
    for i in range(40):
        g = helpers.random_graph(rng, max_vertices=30, max_edges=150)
        ast = helpers.random_ast(rng, unknown_label="zz")
        n = ref_compile(ast, g.label_ids)
        source = rng.randrange(g.num_vertices)
        out.append(instance(g, n, source, f"engine_random_15/{i}"))
    # test_acceptance.py:60-84
    rng = random.Random(0xC1)
    for i in range(500):
        g = helpers.random_graph(rng, max_vertices=50, max_labels=4, max_edges=300)
        ast = helpers.random_ast(rng, labels="abcd", max_depth=4, unknown_label="zz")
        source = rng.randrange(g.num_vertices)
        n = ref_compile(ast, g.label_ids)
        out.append(instance(g, n, source, f"acceptance_c1/{i}"))
    # test_acceptance.py:92-112 (SDR duality)
    rng = random.Random(0xC2)
    for i in range(100):
        g = helpers.random_graph(rng, max_vertices=12, max_labels=4, max_edges=60)
        ast = helpers.random_ast(rng, max_depth=3)
        n = ref_compile(ast, g.label_ids)
        v = rng.randrange(g.num_vertices)
        opts = EngineOptions(timeout=math.inf)
        sdr = eval_sdr(g, n, v, opts)
        by_hand = sorted(u for u in range(g.num_vertices)
                         if v in eval_ssr(g, n, u, opts).reachable)
        assert sorted(sdr.reachable) == by_hand
        d = instance(g, n, v, f"acceptance_c2/{i}")
        d["sdr_expected"] = sorted(sdr.reachable)
        d["sdr_iterations"] = sdr.iterations
        out.append(d)
    # test_acceptance.py:141-153 (a* contains the source)
    rng = random.Random(0xC4)
    ast = parse_query("a*")
    for i in range(100):
        g = helpers.random_graph(rng, max_vertices=40, max_edges=150)
        source = rng.randrange(g.num_vertices)
        n = ref_compile(ast, g.label_ids)
        out.append(instance(g, n, source, f"acceptance_c4/{i}"))
    # test_engine.py:269-279 (hybrid thresholds)
    rng = random.Random(9)
    for i in range(15):
        g = helpers.random_graph(rng, max_vertices=20, max_edges=80)
        pattern = helpers.random_ast(rng, max_depth=3)
        n = ref_compile(pattern, g.label_ids)
        source = rng.randrange(g.num_vertices)
        d = instance(g, n, source, f"hybrid_9/{i}")
        d["threshold_iterations"] = {
            str(t): eval_ssr_hybrid(g, n, source, EngineOptions(switch_threshold=t)).iterations
            for t in (0, 3, math.inf)
        }
        out.append(d)
    out.extend(known_answers())
    return out


def ast_json(node):
    kind = type(node).__name__
    if kind == "Label":
        return {"k": "label", "name": node.name, "inv": bool(node.inverted)}
    if kind in ("Concat", "Alt"):
        return {"k": kind.lower(), "c": [ast_json(c) for c in node.children]}
    return {"k": kind.lower(), "c": ast_json(node.child)}


def plan_record(g, ast, vertex, tag):
    opts = EngineOptions(timeout=math.inf)
    src = eval_plan(g, ast, ("source", vertex), opts)
    dst = eval_plan(g, ast, ("destination", vertex), opts)
    return {"tag": tag, "graph": graph_json(g), "ast": ast_json(ast), "vertex": vertex,
            "source": {"reach": sorted(src.reachable), "iterations": src.iterations},
            "destination": {"reach": sorted(dst.reachable), "iterations": dst.iterations}}


def gen_plan():
    """eval_plan on the RNG streams of test_engine.py:403-415 (seed 15) and
    test_acceptance.py:60-84 (seed 0xC1, first 200), replayed call for call,
    plus the plan-specific cases of test_engine.py:122-153."""
    out = []
    rng = random.Random(15)
    for i in range(40):
        g = helpers.random_graph(rng, max_vertices=30, max_edges=150)
        ast = helpers.random_ast(rng, unknown_label="zz")
        ref_compile(ast, g.label_ids)
        source = rng.randrange(g.num_vertices)
        out.append(plan_record(g, ast, source, f"engine_random_15/{i}"))
    rng = random.Random(0xC1)
    for i in range(200):
        g = helpers.random_graph(rng, max_vertices=50, max_labels=4, max_edges=300)
        ast = helpers.random_ast(rng, labels="abcd", max_depth=4, unknown_label="zz")
        source = rng.randrange(g.num_vertices)
        out.append(plan_record(g, ast, source, f"acceptance_c1/{i}"))
    for tag, text, q, v in [
        ("chain a b c", "0\ta\t1\n1\tb\t2\n2\tc\t3\n", "a b c", "0"),      # test_engine.py:126-131
        ("chain a b c back", "0\ta\t1\n1\tb\t2\n2\tc\t3\n", "a b c", "3"),
        ("star identity", "0\tb\t1\n", "a*", "1"),                                 # :134-137
        ("nested star", "0\ta\t1\n1\tb\t1\n1\ta\t2\n2\tc\t3\n", "(a b*)* c", "0"),  # :140-146
        ("a* no edges", "0\tb\t1\n", "a*", "0"),                                   # test_engine.py:91
    ]:
        g = helpers.load_text(text)
        out.append(plan_record(g, parse_query(q), g.vertex_index(v), f"known/{tag}"))
    return out


def gen_steps():
    """step_update (engine.py:127-138) on the RNG stream of
    test_engine.py:318-329 (seed 12: single-pair frontier, empty P) and on
    random frontiers / visited sets (seed 0x57)."""
    out = []
    rng = random.Random(12)
    for i in range(20):
        g = helpers.random_graph(rng, max_vertices=15, max_edges=60)
        n = ref_compile(helpers.random_ast(rng, max_depth=3), g.label_ids)
        m = SparseBoolMatrix.from_pairs(n.nstates, g.num_vertices, [(0, rng.randrange(g.num_vertices))])
        pm = SparseBoolMatrix.zero(n.nstates, g.num_vertices)
        r = step_update(m, pm, g, n, EngineOptions())
        out.append({"tag": f"orders_12/{i}", "graph": graph_json(g), "nfa": nfa_json(n),
                    "m": m.pairs(), "p": pm.pairs(), "expected": r.pairs()})
    rng = random.Random(0x57)
    for i in range(80):
        g = helpers.random_graph(rng, max_vertices=30, max_edges=150)
        n = ref_compile(helpers.random_ast(rng, unknown_label="zz"), g.label_ids)
        allp = [(q, v) for q in range(n.nstates) for v in range(g.num_vertices)]
        mp = [x for x in allp if rng.random() < 0.15]
        pp = [x for x in allp if rng.random() < 0.3]
        m = SparseBoolMatrix.from_pairs(n.nstates, g.num_vertices, mp)
        pm = SparseBoolMatrix.from_pairs(n.nstates, g.num_vertices, pp)
        r = step_update(m, pm, g, n, EngineOptions())
        out.append({"tag": f"random_57/{i}", "graph": graph_json(g), "nfa": nfa_json(n),
                    "m": m.pairs(), "p": pm.pairs(), "expected": r.pairs()})
    return out


def known_answers():
    triangle = "3\ta\t4\n4\ta\t3\n3\tb\t5\n"
    cases = [
        ("triangle a* b from 3", triangle, "a* b", "3"),           # test_engine.py:103-110
        ("triangle a* from 3", triangle, "a*", "3"),               # :113-117
        ("triangle a* from 4", triangle, "a*", "4"),
        ("triangle a* from 5", triangle, "a*", "5"),
        ("absent label", "1\ta\t2\n", "b", "1"),                   # :120-124
        ("self loop a*", "0\ta\t0\n", "a*", "0"),                  # :127-134
        ("no a-edges a*", "0\tb\t1\n", "a*", "0"),
        ("chain a+", "v0\ta\tv1\nv1\ta\tv2\n", "a+", "v0"),        # :147-154
        ("inverse a ^a", "1\ta\t2\n3\ta\t2\n", "a ^a", "1"),        # :157-165
        ("sdr single edge b", "3\tb\t5\n", "b", "3"),              # :213-217 (ssr side)
        ("chain a b c", "0\ta\t1\n1\tb\t2\n2\tc\t3\n", "a b c", "0"),
        ("nested star", "0\ta\t1\n1\tb\t1\n1\ta\t2\n2\tc\t3\n", "(a b*)* c", "0"),
        ("41-vertex chain a*", "".join(f"{i}\ta\t{i + 1}\n" for i in range(40)), "a*", "0"),
    ]
    out = []
    for name, text, pattern, src_name in cases:
        g = helpers.load_text(text)
        n = ref_compile(parse_query(pattern), g.label_ids)
        d = instance(g, n, g.vertex_index(src_name), f"known/{name}")
        d["expected_names"] = sorted(g.vertices[v] for v in d["expected"])
        out.append(d)
    return out


# ---------------------------------------------------------------------------
# config queries and full-size goldens
# ---------------------------------------------------------------------------


def config_automata():
    from paper_2412_10287_b200 import datagen as D

    out = {}
    for cfg, c in D.CONFIGS.items():
        names = D.rank_names(c["nl"], c["names"])
        labels = {nm: i for i, nm in enumerate(names)}
        for q in c["queries"]:
            for minimize in (True, False):
                n = ref_compile(parse_query(q), labels, minimize=minimize)
                out.setdefault(cfg, {})[f"{q}|{'min' if minimize else 'raw'}"] = nfa_json(n)
    return out


def ref_graph_from_synthetic(sg, used_labels):
    """Reference LabeledGraph over the synthetic arrays; labels the query
    does not use are left empty (result-identical: _label_pairs only touches
    alphabet labels, engine.py:99-102)."""
    nv = sg.nv
    fwd = []
    for l in range(sg.nl):
        if l in used_labels:
            sel = sg.lab == l
            fwd.append(SparseBoolMatrix.from_coo(nv, nv, sg.src[sel].astype(np.int64),
                                                 sg.dst[sel].astype(np.int64)))
        else:
            fwd.append(SparseBoolMatrix.zero(nv, nv))
    return RefGraph([str(i) for i in range(nv)], list(sg.label_names), fwd)


def pack_reach(reachable, nv):
    v = np.zeros(nv, dtype=np.uint8)
    v[list(reachable)] = 1
    return base64.b64encode(np.packbits(v, bitorder="little").tobytes()).decode()


def reach_digest(reachable, nv):
    """sha256 of the little-endian packed answer bitmap (tests/fixtures.py reach_sha256)."""
    import hashlib

    v = np.zeros(nv, dtype=np.uint8)
    v[list(reachable)] = 1
    return hashlib.sha256(np.packbits(v, bitorder="little").tobytes()).hexdigest()


def gen_config(cfg, sources=None, queries=None, minimize=True, count=None):
    from paper_2412_10287_b200 import datagen as D

    t = time.time()
    sg = D.generate(cfg)
    print(f"[{cfg}] generated {sg.ne} edges in {time.time() - t:.1f}s", flush=True)
    c = D.CONFIGS[cfg]
    names = D.rank_names(c["nl"], c["names"])
    full_digest = sg.digest()
    srcs0 = sources if sources is not None else D.pick_sources(sg, cfg, count=count)
    if cfg == "cfg4":
        # 2,000 labels x 90M vertices cannot be a reference LabeledGraph (one
        # int64 indptr per label and direction: 2.6 TiB).
        # The queries use only the 4 most frequent labels (indices 0..3), and
        # _label_pairs touches only alphabet labels (engine.py:99-102): a graph
        # of those 4 labels is result-identical.
        keep = sg.lab < 4
        sg.src, sg.dst, sg.lab = sg.src[keep], sg.dst[keep], sg.lab[keep]
        sg.label_names = sg.label_names[:4]
        names = names[:4]
        print(f"[{cfg}] kept the 4 query labels: {sg.ne} edges", flush=True)
    labels = {nm: i for i, nm in enumerate(names)}
    srcs = srcs0
    records = []
    for q in (queries or c["queries"]):
        n = ref_compile(parse_query(q), labels, minimize=minimize)
        used = {k[0] for k in n.alphabet}
        t = time.time()
        g = ref_graph_from_synthetic(sg, used)
        print(f"[{cfg}] reference graph for {q!r} in {time.time() - t:.1f}s", flush=True)
        for s in srcs:
            t = time.time()
            res = eval_ssr(g, n, s, EngineOptions(timeout=math.inf))
            t_h = time.time() - t
            t = time.time()
            masked = eval_ssr_masked(g, n, s, EngineOptions(timeout=math.inf))
            t_m = time.time() - t
            assert masked.reachable == res.reachable
            rec_bits = {"reach_bits": pack_reach(res.reachable, sg.nv)} if sg.nv <= 20_000_000 else \
                {"reach_sha256": reach_digest(res.reachable, sg.nv)}  # cfg4: 11 MB per answer otherwise
            records.append({
                "query": q, "minimize": minimize, "source": s, "nfa": nfa_json(n),
                "reach_count": len(res.reachable), **rec_bits,
                "iterations": {"hybrid": res.iterations, "masked": masked.iterations},
                "ref_seconds": {"hybrid": t_h, "masked": t_m},
            })
            print(f"[{cfg}] {q!r} src {s}: reach {len(res.reachable)} it {res.iterations} "
                  f"hybrid {t_h:.2f}s masked {t_m:.2f}s", flush=True)
        del g
    return {"config": cfg, "nv": sg.nv, "ne": sg.ne, "digest": full_digest, "records": records,
            "labels_kept": len(names)}


def gen_desk():
    """The reference's desk-scale benchmark analogue (test_acceptance.py:238-335,
    criterion 7) and its determinism bytes (criterion 8, :338-369): the same
    generated graph (cli.generate_edges, seed 0xBE, 1e5 vertices, ~1e6 edges
    with the test's label skew) and the same 1,000-entry workload (rng 0xC7:
    10 families x {ssr, sdr} x 50 endpoints), evaluated by the reference with
    each SSR algorithm.  Writes the graph in index space (desk_graph.npz) and
    per entry the answer count, a sha256 of the sorted answer ids and every
    algorithm's iteration count (desk_bench.json.gz)."""
    import hashlib
    import io

    import test_acceptance as TA
    from rpq.cli import generate_edges, parse_workload
    from rpq.query_compiler import reverse as ref_reverse

    buf = io.StringIO()
    generate_edges(TA._NUM_VERTICES, sorted(TA._desk_scale_counts().items()), 0xBE, buf)
    graph = helpers.load_text(buf.getvalue())
    rng = random.Random(0xC7)
    lines = []
    for fam, pattern in enumerate(TA._QUERY_FAMILIES, start=1):
        for mode in ("ssr", "sdr"):
            for k in range(TA._ENDPOINTS_PER_COMBO):
                endpoint = rng.choice(graph.vertices)
                lines.append(f"q{fam:02d}-{mode}-{k:02d}\t{mode}\t{endpoint}\t{pattern}")
    entries = parse_workload(io.StringIO("\n".join(lines) + "\n"))
    arrays = {"nv": np.array([graph.num_vertices], dtype=np.int64)}
    for l in range(graph.num_labels):
        f = graph.forward[l]
        arrays[f"indptr_{l}"] = np.asarray(f.indptr, dtype=np.int32)
        arrays[f"indices_{l}"] = np.asarray(f.indices, dtype=np.int32)
    np.savez_compressed(os.path.join(HERE, "desk_graph.npz"), **arrays)
    autos = {pattern: nfa_json(ref_compile(parse_query(pattern), graph.label_ids))
             for pattern in TA._QUERY_FAMILIES}
    rows = []
    chunks = []
    t = time.time()
    for e in entries:
        n = ref_compile(parse_query(e.pattern), graph.label_ids)
        v = graph.vertex_index(e.endpoint)
        nn = n if e.mode == "ssr" else ref_reverse(n)
        its = {}
        reach = None
        for alg, fn in (("masked", eval_ssr_masked), ("no_mask", eval_ssr_no_mask),
                        ("hybrid", eval_ssr_hybrid)):
            r = fn(graph, nn, v, EngineOptions(timeout=60.0))
            its[alg] = r.iterations
            assert reach is None or reach == r.reachable
            reach = r.reachable
        # criterion 8's bytes: eval_ssr / eval_sdr with the hybrid default
        h = (eval_ssr if e.mode == "ssr" else eval_sdr)(graph, n, v, EngineOptions(algorithm="hybrid",
                                                                                   timeout=60.0))
        assert h.reachable == reach
        ids = ",".join(str(x) for x in sorted(reach))
        chunks.append(f"{e.id}:{ids}")
        rows.append({"id": e.id, "mode": e.mode, "pattern": e.pattern, "vertex": v,
                     "count": len(reach), "sha256": hashlib.sha256(ids.encode()).hexdigest(),
                     "iterations": its})
    c8 = hashlib.sha256("\n".join(chunks).encode()).hexdigest()
    print(f"desk bench: {len(rows)} entries in {time.time() - t:.1f}s; criterion-8 sha256 {c8}")
    return {"nv": graph.num_vertices, "labels": list(graph.labels), "automata": autos,
            "entries": rows, "criterion8_sha256": c8,
            "num_edges": int(sum(graph.forward[l].nnz for l in range(graph.num_labels)))}


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "random"
    if what == "random":
        inst = gen_random()
        path = os.path.join(HERE, "reference_instances.json.gz")
        with gzip.open(path, "wt") as fh:
            json.dump(inst, fh)
        print(f"wrote {len(inst)} instances to {path}")
    elif what == "plan":
        out = gen_plan()
        path = os.path.join(HERE, "plan.json.gz")
        with gzip.open(path, "wt") as fh:
            json.dump(out, fh)
        print(f"wrote {len(out)} plan cases to {path}")
    elif what == "desk":
        out = gen_desk()
        path = os.path.join(HERE, "desk_bench.json.gz")
        with gzip.open(path, "wt") as fh:
            json.dump(out, fh)
        print(f"wrote {path}")
    elif what == "steps":
        out = gen_steps()
        path = os.path.join(HERE, "step_update.json.gz")
        with gzip.open(path, "wt") as fh:
            json.dump(out, fh)
        print(f"wrote {len(out)} step cases to {path}")
    elif what == "extra":
        labels = {c: i for i, c in enumerate("abcdefgh")}
        queries = ["^a (b|c)* d", "a ^b* c", "a b*", "(a|^b)* c+", "(a ^a)* (b | c ^d)*",
                   "a*", "a+ b", "(a|b|c|d)*", "a ^b c*", "(a b)* | (c ^d)+ e?"]
        out = {q: nfa_json(ref_compile(parse_query(q), labels)) for q in queries}
        path = os.path.join(HERE, "extra_automata.json")
        with open(path, "w") as fh:
            json.dump(out, fh, indent=1)
        print(f"wrote {path}")
    elif what == "automata":
        path = os.path.join(ROOT, "paper_2412_10287_b200", "data", "config_automata.json")
        os.makedirs(os.path.dirname(path), exist_ok=True)
        with open(path, "w") as fh:
            json.dump(config_automata(), fh, indent=1)
        print(f"wrote {path}")
    elif what == "config":
        args = sys.argv[2:]
        raw = "--raw" in args
        args = [a for a in args if a != "--raw"]
        for spec in args:
            spec, _, cnt = spec.partition("#")
            cfg, _, srcs = spec.partition(":")
            sources = [int(x) for x in srcs.split(",")] if srcs else None
            d = gen_config(cfg, sources=sources, minimize=not raw,
                           count=int(cnt) if cnt else None)
            suffix = "_raw" if raw else ""
            path = os.path.join(HERE, f"{cfg}{suffix}.json.gz")
            with gzip.open(path, "wt") as fh:
                json.dump(d, fh)
            print(f"wrote {path}")
    else:
        raise SystemExit(f"unknown target {what}")


if __name__ == "__main__":
    main()
