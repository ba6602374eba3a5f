"""Where the end-to-end time of eval_ssr goes, per source, without mixing
output modes on one handle (each mode keeps its own captured graph):

  eval_ssr         the public call (pinned answer buffer from the pool)
  fused            rpq_query_eval on a pooled pinned buffer (C only)
  enqueue / wait   rpq_query_run + rpq_query_wait split of the same
  device_ms        CUDA events around the run's graph (H2D inputs, kernel,
                   zero-copy outputs)

    python tools/e2e_split.py [cfg3] [source ...]
"""
import ctypes
import json
import math
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import paper_2412_10287_b200 as P
    from paper_2412_10287_b200 import _lib, datagen
    from paper_2412_10287_b200.engine import _ANSWERS, _table_for
    from paper_2412_10287_b200.graph import device_graph

    cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
    sg = datagen.generate(cfg)
    g = sg.labeled_graph()
    srcs = [int(x) for x in sys.argv[2:]] or datagen.pick_sources(sg, cfg, count=2)
    autos = json.load(open(os.path.join(ROOT, "paper_2412_10287_b200", "data", "config_automata.json")))
    n = P.Automaton.from_json(autos[cfg][datagen.CONFIGS[cfg]["queries"][0] + "|min"])
    opts = P.EngineOptions(timeout=math.inf)
    lib = _lib.engine()
    nwords = (g.num_vertices + 31) // 32
    for s in srcs:
        T = {}
        for _ in range(5):
            P.eval_ssr(g, n, s, opts)
        for _ in range(20):
            t = time.perf_counter()
            r = P.eval_ssr(g, n, s, opts)
            T.setdefault("eval_ssr", []).append(time.perf_counter() - t)
            del r
        dg = device_graph(g)
        table = _table_for(n, g.num_labels)
        q = dg.acquire_query(table)
        buf = _ANSWERS.take(nwords)
        st = _lib.RpqStats()
        for _ in range(20):
            t = time.perf_counter()
            rc = lib.rpq_query_eval(q, s, -1.0, 0, 0, 4.0, 1, ctypes.byref(st), buf.ctypes.data, nwords)
            T.setdefault("fused", []).append(time.perf_counter() - t)
            assert rc == 0, _lib.last_error()
            T.setdefault("device_ms", []).append(st.device_ms / 1e3)
        for _ in range(20):
            lib.rpq_query_set_output(q, 0)
            t = time.perf_counter()
            lib.rpq_query_run(q, s, -1.0, None)
            t1 = time.perf_counter()
            lib.rpq_query_wait(q, ctypes.byref(st))
            t2 = time.perf_counter()
            T.setdefault("enqueue(no answer)", []).append(t1 - t)
            T.setdefault("wait(no answer)", []).append(t2 - t1)
            T.setdefault("device_ms(no answer)", []).append(st.device_ms / 1e3)
        dg.release_query(table, q)
        print(json.dumps({"config": cfg, "source": s, "reach": int(st.reach_count),
                          **{k: round(1e6 * statistics.median(v), 1) for k, v in T.items()}}))


if __name__ == "__main__":
    main()
