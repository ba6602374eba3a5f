"""Per-CTA phase stamps of one query (RPQ_TUNE_TRACE): for every level, the
spread over CTAs of level start, plan-epoch end, expansion end and barrier
exit -- where the level's time goes (critical CTA vs everyone waiting).

    python tools/trace_probe.py [cfg2] [--levels 16] [--no-flush]
"""
import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="cfg2")
    ap.add_argument("--levels", type=int, default=16)
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--direction", default="auto")
    ap.add_argument("--query", type=int, default=0, help="index into the config's query templates")
    ap.add_argument("--max-degree", action="store_true", help="source = max out-degree vertex (bench.py's)")
    ap.add_argument("--source", type=int, default=None, help="explicit source vertex")
    args = ap.parse_args()
    import numpy as np
    import torch

    import paper_2412_10287_b200 as P
    from paper_2412_10287_b200 import _lib, datagen

    autos = json.load(open(os.path.join(ROOT, "paper_2412_10287_b200", "data", "config_automata.json")))
    c = datagen.CONFIGS[args.config]
    sg = datagen.generate(args.config)
    g = sg.labeled_graph()
    n = P.Automaton.from_json(autos[args.config][c["queries"][args.query] + "|min"])
    if args.source is not None:
        src = args.source
    elif args.max_degree:
        src = int(np.argmax(sg.out_degree()))
    else:
        src = int(datagen.pick_sources(sg, args.config, count=1)[0])
    pq = P.PreparedQuery(g, n)
    pq.set_options(direction=args.direction)
    lib = _lib.engine()
    assert lib.rpq_query_set_tuning(pq.q, _lib.TUNE_TRACE, float(args.levels)) == 0, _lib.last_error()
    s = torch.cuda.Stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for rep in range(4):
        with torch.cuda.stream(s):
            if not args.no_flush:
                flush.fill_(rep)
        pq.launch(src, -1.0, s.cuda_stream)
        st = pq.wait()
    grid = ctypes.c_int32()
    n_ = args.levels * 160 * 8
    buf = np.zeros(n_, dtype=np.uint64)
    assert lib.rpq_query_copy_trace(pq.q, _lib.ptr(buf, ctypes.c_uint64), n_, ctypes.byref(grid)) == 0
    G = grid.value
    tr = buf[: args.levels * G * 8].reshape(args.levels, G, 8).astype(np.float64) / 1e3
    d = st.to_dict()
    print(json.dumps({"config": args.config, "device_ms": st.device_ms, "iterations": st.iterations,
                      "dirs": d["level_dir"], "new": d["level_new"]}))
    for L in range(args.levels):
        t = tr[L]
        if not t[:, 0].any():
            # the row of the deciding level that ended the loop: its decision
            # stamps (5-7) and the epilogue's (1: entered, 2: projection
            # written, 3: answer transport written, 4: done)
            ep = {"L": L, "epilogue": True,
                  "dec_enter": (tr[L, :, 6].min(), tr[L, :, 6].max()),
                  "dec_end": (tr[L, :, 7].min(), tr[L, :, 7].max())}
            for k, name in ((1, "entered"), (2, "projected"), (3, "transport"), (4, "done")):
                col = t[:, k]
                if col.any():
                    ep[name] = (col.min(), col.max())
            print(json.dumps({k: [round(float(x), 2) for x in v] if isinstance(v, tuple) else v
                              for k, v in ep.items()}))
            break
        plan = t[:, 1]
        row = {"L": L, "dir": d["level_dir"][L] if L < len(d["level_dir"]) else None,
               "start_min": t[:, 0].min(), "start_max": t[:, 0].max(),
               "plan_max": plan.max() if plan.any() else None,
               "work_min": t[:, 2].min(), "work_med": float(np.median(t[:, 2])), "work_max": t[:, 2].max(),
               "flush_max": t[:, 4].max(),
               "dec_enter": (tr[L, :, 6].min(), tr[L, :, 6].max()),
               "dec_loaded": (tr[L, :, 5].min(), tr[L, :, 5].max()),
               "dec_end": (tr[L, :, 7].min(), tr[L, :, 7].max()),
               "bar_min": t[:, 3].min(), "bar_max": t[:, 3].max(),
               "slowest_cta": int(np.argmax(t[:, 2]))}
        rnd = (lambda v: round(float(v), 2) if isinstance(v, (float, np.floating)) else
               [round(float(x), 2) for x in v] if isinstance(v, tuple) else v)
        print(json.dumps({k: rnd(v) for k, v in row.items()}))
    pq.close()


if __name__ == "__main__":
    main()
