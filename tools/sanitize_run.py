"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): every device kernel of the engine on inputs that finish quickly
under instrumentation, each answer checked against the CPU oracle.

    compute-sanitizer --tool memcheck python tools/sanitize_run.py [--quick]

Covers: the single-CTA kernel (cfg1), the grid kernel under auto/push/pull
(cfg1 forced to the grid; a scale-14 R-MAT with the cfg2 query), step mode
(step_update), the bit-sliced batch kernel (32 and 40 sources), device ingest
(COO -> per-label CSR/CSC) and the merged-slot build ((a|b|c|d)*)."""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    args = ap.parse_args()
    import numpy as np

    import paper_2412_10287_b200 as P
    from paper_2412_10287_b200 import datagen
    from oracle import OracleGraph, OracleQuery, oracle_bfs

    autos = json.load(open(os.path.join(ROOT, "paper_2412_10287_b200", "data", "config_automata.json")))
    extra = json.load(open(os.path.join(ROOT, "tests", "golden", "extra_automata.json")))
    checked = 0

    def check(sg, g, nj, sources, kernels=("auto", "grid"), directions=("auto", "push", "pull")):
        nonlocal checked
        og = OracleGraph(sg.nv, sg.nl, sg.src, sg.dst, sg.lab)
        oq = OracleQuery(nj, sg.nl)
        n = P.Automaton.from_json(nj)
        for s in sources:
            want, st = oracle_bfs(og, oq, s)
            for kernel in kernels:
                for d in directions:
                    r = P.eval_ssr(g, n, s, P.EngineOptions(timeout=math.inf, kernel=kernel, direction=d))
                    assert np.array_equal(r.reach, want), (s, kernel, d)
                    assert r.iterations == st["iterations"], (s, kernel, d)
                    checked += 1
        rows = P.eval_ssr_batch(g, n, sources, P.EngineOptions(timeout=math.inf))
        for s, row in zip(sources, rows):
            assert np.array_equal(row, oracle_bfs(og, oq, s)[0]), ("batch", s)
            checked += 1

    # cfg1: single-CTA kernel and the grid kernel
    sg = datagen.generate("cfg1")
    g = sg.labeled_graph()
    check(sg, g, autos["cfg1"]["a b*|min"], [0, 1, 77] if not args.quick else [0])
    # R-MAT scale 14 with the cfg2 query (host CSR upload path)
    sg = datagen.generate("cfg2", scale=14)
    g = sg.labeled_graph()
    srcs = [int(v) for v in np.argsort(-sg.out_degree(), kind="stable")[:2]]
    check(sg, g, autos["cfg2"]["a ^b* c|min"], srcs)
    # 40 sources: two batch launches, the second partial
    n = P.Automaton.from_json(autos["cfg2"]["a ^b* c|min"])
    og = OracleGraph(sg.nv, sg.nl, sg.src, sg.dst, sg.lab)
    oq = OracleQuery(autos["cfg2"]["a ^b* c|min"], sg.nl)
    many = [int(s) for s in datagen.pick_sources(sg, "cfg3", count=40)]
    rows = P.eval_ssr_batch(g, n, many, P.EngineOptions(timeout=math.inf))
    for s, row in zip(many, rows):
        assert np.array_equal(row, oracle_bfs(og, oq, s)[0]), ("batch40", s)
        checked += 1
    # device ingest (COO) and merged slots: (a|b|c|d)* and a two-way shape
    dg_graph = P.LabeledGraph.from_coo(sg.nv, sg.label_names, sg.src, sg.dst, sg.lab)
    for q in ("(a|b|c|d)*", "a ^b c*", "(a ^a)* (b | c ^d)*"):
        nj = extra[q]
        check(sg, dg_graph, nj, srcs[:1], kernels=("grid",), directions=("auto",))
    # step mode: one step from the seed
    from paper_2412_10287_b200.graph import CsrMatrix

    nstates = n.nstates
    m = CsrMatrix.from_pairs(nstates, sg.nv, [(0, srcs[0])])
    out = P.step_update(m, m, g, n, P.EngineOptions())
    assert out.nnz >= 0
    checked += 1
    print(json.dumps({"sanitize_run": "ok", "checks": checked}))


if __name__ == "__main__":
    main()
