"""Cost of one device step (rpq_query_step_device, the partitioned
evaluator's per-level kernel) on cfg3's graph: empty M, a 1-vertex M, and a
dense M; chained without host syncs (step_begin .. step_end) and one by one.

    python tools/step_probe.py
"""
import ctypes
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    import paper_2412_10287_b200 as P
    from paper_2412_10287_b200 import _lib, datagen
    from paper_2412_10287_b200.partition import DeviceStep

    sg = datagen.generate("cfg3")
    g = sg.labeled_graph()
    nj = json.load(open(os.path.join(ROOT, "paper_2412_10287_b200", "data", "config_automata.json")))["cfg3"]["^a (b|c)* d|min"]
    n = P.Automaton.from_json(nj)
    step = DeviceStep(g, n, "cuda:0")
    W = step.row_words
    m = torch.zeros((n.nstates, W), dtype=torch.int32, device="cuda")
    p = torch.zeros_like(m)
    out = torch.zeros_like(m)
    s = torch.cuda.Stream()
    res = {}
    for name, fill in (("empty", None), ("one", 10754584), ("dense", "dense")):
        m.zero_()
        p.zero_()
        if fill == "dense":
            m[1, : W // 4] = -1
        elif fill is not None:
            m[0, fill >> 5] = 1 << (fill & 31)
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            p.zero_()
            torch.cuda.synchronize()
            t = time.perf_counter()
            step(m, p, out, s.cuda_stream)
            ms = step.finish()
            ts.append((time.perf_counter() - t, ms))
        res[name] = {"wall_us": 1e6 * float(np.median([a for a, _ in ts])), "device_us": 1e3 * float(np.median([b for _, b in ts]))}
        # a chain of 8 steps without host syncs
        torch.cuda.synchronize()
        step.begin(s.cuda_stream)
        t = time.perf_counter()
        for _ in range(8):
            step(m, p, out, s.cuda_stream)
        cnt = step.count()
        res[name]["chain8_wall_us_per_step"] = 1e6 * (time.perf_counter() - t) / 8
    print(json.dumps(res))


if __name__ == "__main__":
    main()
