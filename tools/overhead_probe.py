"""Measure the engine's fixed costs on the device: an empty query (seed only),
and a long chain (one vertex per BFS level), to isolate per-level overhead."""
import json
import math
import sys
import time

sys.path.insert(0, ".")
import numpy as np

import paper_2412_10287_b200 as P


def timed(pq, src, reps=20):
    ts = []
    for _ in range(reps):
        pq.launch(src)
        st = pq.wait()
        ts.append(st.device_ms)
    return float(np.median(ts)), st


def main():
    out = {}
    for n in (1000, 4000):
        g = P.LabeledGraph.from_edges(n + 1, ["a"], [(i, 0, i + 1) for i in range(n)])
        a = P.Automaton.build(1, {(0, False): [(0, 0)]}, [0], [0])
        pq = P.PreparedQuery(g, a)
        for d in ("push", "pull"):
            pq.set_options(direction=d)
            ms, st = timed(pq, 0)
            out[f"chain{n}_{d}"] = {"ms": ms, "iterations": st.iterations,
                                    "us_per_level": 1e3 * ms / st.iterations,
                                    "level_us": [t / 1e3 for t in st.level_ns[:8]],
                                    "work_us": [t / 1e3 for t in st.work_ns[:8]],
                                    "bar_us": [t / 1e3 for t in st.bar_ns[:8]]}
        # empty: source has no out-edges
        pq.set_options(direction="push")
        ms, st = timed(pq, n)
        out[f"chain{n}_from_sink"] = {"ms": ms, "iterations": st.iterations}
        pq.close()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
