"""Measure every BASELINE.json configuration on one GPU: for each query of the
config and each of its sources, one untimed run for the exact work counts,
then `--reps` device-timed runs (CUDA events, L2 flushed before each).

    python tools/config_sweep.py cfg1 cfg2 cfg3 cfg4 cfg5 [--sources 8] [--reps 3]

Prints one JSON object per (config, query): GTEPS = sum TE / sum device time,
per-query latency, the algorithmic bytes of SURVEY.md §8(d) and their
fraction of the measured HBM peak.  Used for profiles/; bench.py is the
contract line (cfg2).
"""

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
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--sources", type=int, default=8)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--raw", action="store_true", help="unminimized automata (cfg5: 17 states)")
    args = ap.parse_args()

    import numpy as np
    import torch

    import paper_2412_10287_b200 as P
    from paper_2412_10287_b200 import datagen

    sys.path.insert(0, ROOT)
    from bench import algorithmic_bytes, read_peaks

    autos = json.load(open(os.path.join(ROOT, "paper_2412_10287_b200", "data", "config_automata.json")))
    peak, peak_src = read_peaks()
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for cfg in args.configs:
        t = time.time()
        sg = datagen.generate(cfg)
        gen_s = time.time() - t
        g = sg.labeled_graph()
        c = datagen.CONFIGS[cfg]
        if c["sources"] in ("zero", "max_out_degree"):
            sources = datagen.pick_sources(sg, cfg)
        else:
            sources = datagen.pick_sources(sg, cfg, count=args.sources)
        for query in c["queries"]:
            nj = autos[cfg][f"{query}|{'raw' if args.raw else 'min'}"]
            n = P.Automaton.from_json(nj)
            t = time.time()
            pq = P.PreparedQuery(g, n)
            upload_s = time.time() - t
            te_sum = bytes_sum = 0
            ms_sum = 0.0
            lat = []
            levels = []
            reach = []
            for s in sources:
                pq.set_options(count_te=True)
                pq.launch(s, -1.0, stream.cuda_stream)
                st = pq.wait()
                per_state = pq.visited_counts()
                outdeg = np.bincount(pq.table.t_src, minlength=pq.table.nstates)
                x = int((per_state * outdeg).sum())
                b = algorithmic_bytes(int(st.te), x, int(st.visited_pairs), int(st.iterations),
                                      pq.table.nstates, sg.nv)
                pq.set_options(count_te=False)
                times = []
                for _ in range(args.reps):
                    flush.fill_(1)
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    pq.launch(s, -1.0, stream.cuda_stream)
                    e1.record(stream)
                    pq.wait()
                    torch.cuda.synchronize()
                    times.append(e0.elapsed_time(e1))
                ms = float(np.median(times))
                te_sum += int(st.te) * 1
                bytes_sum += b
                ms_sum += ms
                lat.append(ms)
                levels.append(int(st.iterations))
                reach.append(int(st.reach_count))
            pq.close()
            out = {
                "config": cfg, "query": query, "states": n.nstates, "vertices": sg.nv, "edges": sg.ne,
                "sources": len(sources), "gteps": te_sum / (ms_sum / 1e3) / 1e9 if ms_sum else None,
                "latency_ms_median": float(np.median(lat)), "latency_ms_max": float(np.max(lat)),
                "te_total": te_sum, "iterations": levels, "reach": reach,
                "roofline": {"achieved_gbs": bytes_sum / (ms_sum / 1e3) / 1e9 if ms_sum else None,
                             "peak_gbs": peak, "frac": (bytes_sum / (ms_sum / 1e3) / 1e9) / peak if ms_sum else None,
                             "peak_source": peak_src, "algorithmic_bytes": bytes_sum},
                "generate_s": gen_s, "upload_s": upload_s,
            }
            print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
