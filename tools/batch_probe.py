"""Multi-source throughput: the bit-sliced batch kernel (64 sources per
launch) against the single-source kernel run once per source, on the same
sources of a BASELINE config (default cfg5, 1,024 sources).

    python tools/batch_probe.py [cfg5] [--sources 1024] [--single 64]

Prints one JSON line: GTEPS = sum over sources of TE / device time."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="cfg5")
    ap.add_argument("--sources", type=int, default=1024)
    ap.add_argument("--single", type=int, default=64, help="sources timed on the single-source kernel")
    ap.add_argument("--query", type=int, default=0)
    args = ap.parse_args()

    import numpy as np
    import torch

    import paper_2412_10287_b200 as P
    from paper_2412_10287_b200 import datagen

    autos = json.load(open(os.path.join(ROOT, "paper_2412_10287_b200", "data", "config_automata.json")))
    sg = datagen.generate(args.config)
    g = sg.labeled_graph()
    c = datagen.CONFIGS[args.config]
    query = c["queries"][args.query]
    n = P.Automaton.from_json(autos[args.config][f"{query}|min"])
    srcs = [int(s) for s in datagen.pick_sources(sg, args.config, count=args.sources)]
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    pq = P.PreparedQuery(g, n)
    # batch kernel
    pq.launch_batch(srcs[:64], -1.0, stream.cuda_stream)
    pq.wait_batch()
    te_b = 0
    ms_b = 0.0
    rows_b = 0
    levels = []
    detail = None
    for b0 in range(0, len(srcs), 64):
        with torch.cuda.stream(stream):
            flush.fill_(1)
        pq.launch_batch(srcs[b0:b0 + 64], -1.0, stream.cuda_stream)
        st = pq.wait_batch()
        te_b += int(st.te)
        rows_b += int(st.rows)
        ms_b += float(st.device_ms)
        if detail is None:
            detail = st.to_dict()
        levels.append(int(st.levels))
    # single-source kernel on a prefix of the same sources
    pq.set_options(count_te=True)
    te_s = 0
    ms_s = 0.0
    te_s_prefix_batch = 0
    for s in srcs[: args.single]:
        pq.launch(s, -1.0, stream.cuda_stream)
        st = pq.wait()
        te_s += int(st.te)
    pq.set_options(count_te=False)
    for s in srcs[: args.single]:
        with torch.cuda.stream(stream):
            flush.fill_(1)
        pq.launch(s, -1.0, stream.cuda_stream)
        st = pq.wait()
        ms_s += float(st.device_ms)
    # batch TE over the same prefix (whole batches)
    for b0 in range(0, args.single, 64):
        pq.launch_batch(srcs[b0:b0 + 64], -1.0, stream.cuda_stream)
        te_s_prefix_batch += int(pq.wait_batch().te)
    pq.close()
    out = {
        "config": args.config, "query": query, "sources": len(srcs),
        "batch": {"gteps": te_b / (ms_b / 1e3) / 1e9 if ms_b else None, "te": te_b, "ms_total": ms_b,
                  "ms_per_source": ms_b / len(srcs), "levels": levels[:8],
                  "rows": rows_b, "sharing": te_b / max(rows_b, 1), "first_batch": detail},
        "single": {"sources": args.single, "gteps": te_s / (ms_s / 1e3) / 1e9 if ms_s else None,
                   "te": te_s, "ms_per_source": ms_s / max(args.single, 1)},
        "te_agree_on_prefix": te_s == te_s_prefix_batch,
    }
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
