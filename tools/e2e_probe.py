"""Break down the host-side cost of one eval_ssr call.

    python tools/e2e_probe.py [cfg2] [source]   (default source: the config's first)"""
import json
import math
import sys
import time

sys.path.insert(0, ".")
import ctypes

import numpy as np

import paper_2412_10287_b200 as P
from paper_2412_10287_b200 import _lib, datagen
from paper_2412_10287_b200.engine import _table_for, bits_to_reach
from paper_2412_10287_b200.graph import device_graph

CFG = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
sg = datagen.generate(CFG)
g = sg.labeled_graph()
SRC = int(sys.argv[2]) if len(sys.argv) > 2 else int(datagen.pick_sources(sg, CFG, count=1)[0])
nj = json.load(open("paper_2412_10287_b200/data/config_automata.json"))[CFG][datagen.CONFIGS[CFG]["queries"][0] + "|min"]
n = P.Automaton.from_json(nj)
opts = P.EngineOptions(timeout=math.inf)
for _ in range(5):
    P.eval_ssr(g, n, SRC, opts)
lib = _lib.engine()
T = {}


def tick(k, t):
    T.setdefault(k, []).append(time.perf_counter() - t)


for _ in range(20):
    t = time.perf_counter(); P.eval_ssr(g, n, SRC, opts); tick("eval_ssr total", t)
    t = time.perf_counter(); dg = device_graph(g); tick("device_graph", t)
    t = time.perf_counter(); table = _table_for(n, g.num_labels); tick("table", t)
    t = time.perf_counter(); dg.ensure_labels(table.labels); tick("ensure_labels", t)
    t = time.perf_counter(); q = dg.acquire_query(table); tick("acquire", t)
    t = time.perf_counter(); lib.rpq_query_set_options(q, 0, 0, 4.0); lib.rpq_query_set_output(q, 1); tick("set_opts", t)
    t = time.perf_counter(); lib.rpq_query_run(q, SRC, -1.0, None); tick("run(enqueue)", t)
    tq = time.perf_counter()
    st = _lib.RpqStats()
    t = time.perf_counter(); lib.rpq_query_wait(q, ctypes.byref(st)); tick("wait", t); tick("enqueue->done", tq)
    words = np.empty((g.num_vertices + 31) // 32, dtype=np.uint32)
    t = time.perf_counter(); lib.rpq_query_copy_reach_bits(q, _lib.ptr(words, ctypes.c_uint32), words.size); tick("copy_bits", t)
    t = time.perf_counter(); r = bits_to_reach(words, g.num_vertices); tick("unpack", t)
    tick("device_ms", 0); T["device_ms"][-1] = st.device_ms / 1e3
    dg.release_query(table, q)
    words2 = np.empty((g.num_vertices + 31) // 32, dtype=np.uint32)
    q = dg.acquire_query(table)
    t = time.perf_counter()
    lib.rpq_query_eval(q, SRC, -1.0, 0, 0, 4.0, 1, ctypes.byref(st), _lib.ptr(words2, ctypes.c_uint32), words2.size)
    tick("rpq_query_eval (fused C)", t)
    dg.release_query(table, q)
for k, v in T.items():
    print(f"{k:16s} median {1e6 * float(np.median(v)):9.1f} us")
