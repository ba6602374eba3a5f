"""End-to-end cost of one cfg2 query through the fused C call
(rpq_query_eval: options, run, wait, answer bitmap to the caller) with
RPQ_TUNE_ZERO_COPY off and on, L2 flushed before every call.

    python tools/zc_probe.py [--reps 200]
"""
import argparse
import ctypes
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=200)
    args = ap.parse_args()
    import numpy as np
    import torch

    import paper_2412_10287_b200 as P
    from paper_2412_10287_b200 import _lib, datagen

    autos = json.load(open(os.path.join(ROOT, "paper_2412_10287_b200", "data", "config_automata.json")))
    sg = datagen.generate("cfg2")
    g = sg.labeled_graph()
    n = P.Automaton.from_json(autos["cfg2"]["a ^b* c|min"])
    src = int(np.argmax(sg.out_degree()))
    pq = P.PreparedQuery(g, n)
    lib = _lib.engine()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    words = np.empty((g.num_vertices + 31) // 32, dtype=np.uint32)
    st = _lib.RpqStats()
    out = {}
    ref = None
    for rnd in range(2):
        for zc in (0, 1):
            assert lib.rpq_query_set_tuning(pq.q, _lib.TUNE_ZERO_COPY, float(zc)) == 0, _lib.last_error()
            ts = []
            for k in range(args.reps + 5):
                flush.fill_(k & 0xFF)
                torch.cuda.synchronize()
                t = time.perf_counter()
                rc = lib.rpq_query_eval(pq.q, src, -1.0, 0, 0, 4.0, 1, ctypes.byref(st),
                                        _lib.ptr(words, ctypes.c_uint32), words.size)
                ts.append(time.perf_counter() - t)
                assert rc == 0, _lib.last_error()
            if ref is None:
                ref = words.copy()
            assert np.array_equal(words, ref)
            out[f"zc{zc}_r{rnd}_us"] = round(1e6 * float(np.median(ts[5:])), 1)
    print(json.dumps(out))
    pq.close()


if __name__ == "__main__":
    main()
