#!/usr/bin/env python
"""Benchmark: 2-RPQ product edges traversed per second (GTEPS) and per-query
latency on BASELINE.json's largest single-GPU configuration (configs[2] = cfg3):

  R-MAT scale 24 (16,777,216 vertices), edge factor 16, (0.57, 0.19, 0.19, 0.05),
  self-loops and duplicates removed, 64 Zipf(1.0) labels; two-way query
  ^a (b|c)* d (the reference compiler's minimal 3-state DFA); sources drawn
  uniformly from the vertices with out-degree >= 1 (BASELINE's rule; the first
  8 draws of datagen.pick_sources).  Synthetic, seeded (paper_2412_10287_b200/datagen.py).

A step evaluates every bench source once, one single-source query (seed ->
answer vector ready on the device) per launch.  `value` = sum of the product
edges traversed / sum of the query times, device-timed with CUDA events
around each query on the launching stream (inputs resident in HBM, L2
flushed before every query, outside the events); `e2e` is the same metric
through the public API `eval_ssr` with the automaton sent host->device every
call and the answer read back to the host.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl engine|reference]
                  [--config cfgN] [--sources S]

With N > 1 (torchrun, one rank per GPU) every rank evaluates its own S
sources (the next S draws of the same rule) with no data-path collective
(weak scaling over independent queries).  `--impl reference` times the
reference algorithm's CPU restatement (oracle/rpq_oracle.c oracle_port, the
hybrid loop of engine.py:197-232) on all host cores over the same sources;
rank 0 only.
"""

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))  # checker: cpu_baseline and --impl reference only

METRIC = "2-RPQ edges traversed/sec (GTEPS)"
UNIT = "GTEPS"
CONFIG = "cfg3"
QUERY = "^a (b|c)* d"
WORKLOADS = {
    "cfg1": ("a b*", "cfg1: Erdos-Renyi 10,000 V / 100,000 E, 4 uniform labels, query a b* "
                     "(2-state min DFA), source 0"),
    "cfg2": ("a ^b* c", "cfg2: R-MAT scale 20 (1,048,576 V), edge factor 16, abc=(0.57,0.19,0.19), "
                        "16 Zipf(1.0) labels, query a ^b* c (3-state min DFA), source = max out-degree"),
    "cfg3": ("^a (b|c)* d", "cfg3: R-MAT scale 24 (16,777,216 V), edge factor 16, 64 Zipf(1.0) labels, "
                            "query ^a (b|c)* d (3-state min DFA), sources uniform over out-degree >= 1"),
    "cfg4": ("(a|b|c|d)*", "cfg4: Chung-Lu 90M V / 1.2B raw edges (exponent 2.1), 2,000 Zipf(1.1) labels, "
                           "query (a|b|c|d)* (1-state min DFA), source = max out-degree"),
    "cfg5": ("(a1 a2*) (a3 a4*) (a5 a6*) (a7 a8*) (a9 a10*) (a11 a12*) (a13 a14*) (a15 a16*)",
             "cfg5: R-MAT scale 22, 32 Zipf(1.0) labels, 8-group chain query (9-state min DFA), "
             "source = max out-degree"),
}
WORKLOAD = WORKLOADS[CONFIG][1]
SOURCE_RULE = {
    "cfg1": "vertex 0",
    "cfg2": "highest out-degree vertex (ties: lowest id)",
    "cfg3": "uniform over vertices with out-degree >= 1: datagen.pick_sources draws j = 0.. (seed 103)",
    "cfg4": "uniform over vertices with out-degree >= 1: datagen.pick_sources draws j = 0.. (seed 104)",
    "cfg5": "uniform over vertices with out-degree >= 1: datagen.pick_sources draws j = 0.. (seed 105)",
}
L2_FLUSH_BYTES = 256 << 20


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["engine", "reference"], default="engine")
    ap.add_argument("--mode", choices=["replicas", "partitioned", "batch"], default="replicas",
                    help="replicas: independent single-source queries per rank (default); partitioned: each "
                         "query vertex-partitioned over all ranks (NCCL allgather per level, strong scaling); "
                         "batch: the multi-source kernel over the config's source set, sources sharded over "
                         "ranks (cfg5's 1,024)")
    ap.add_argument("--config", default=CONFIG)
    ap.add_argument("--sources", type=int, default=None,
                    help="sources per rank (uniform-source configs; default 8, batch mode: the config's set)")
    ap.add_argument("--source", type=int, default=None, help="diagnostic: one fixed source instead")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--automaton", choices=["min", "raw"], default="min",
                    help="the reference compiler's minimal DFA (default) or its unminimized automaton")
    ap.add_argument("--direction", choices=["auto", "push", "pull"], default="auto")
    ap.add_argument("--emit-mode", type=int, default=None, help="tuning: 0 inline, 1 plan, 2 adaptive")
    ap.add_argument("--emit-inline-max", type=int, default=None)
    ap.add_argument("--flags", type=int, default=None, help="tuning: push variants (RPQ_TUNE_FLAGS)")
    ap.add_argument("--defer", type=float, default=None, help="tuning: RPQ_TUNE_DEFER factor")
    ap.add_argument("--reorder", action="store_true",
                    help="experiment: relabel vertices by descending total degree before ingest")
    ap.add_argument("--zero-copy", type=int, default=None, choices=[0, 1],
                    help="tuning: RPQ_TUNE_ZERO_COPY (statistics block written straight to pinned host memory)")
    ap.add_argument("--alpha", type=float, default=None, help="tuning: Beamer switch constant (default: engine's)")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-flush", action="store_true", help="keep L2 warm between steps (diagnostic)")
    ap.add_argument("--profile", action="store_true",
                    help="short run for ncu: no e2e leg, no CPU baseline, no clocks")
    return ap.parse_args()


_AUTOMATON_KIND = ["min"]


def load_automaton(config, query):
    """The reference compiler's automaton for the config query: minimal DFA
    (its default), or --automaton raw (minimize=False: cfg5's 17 states)."""
    with open(os.path.join(ROOT, "paper_2412_10287_b200", "data", "config_automata.json")) as fh:
        return json.load(fh)[config][f"{query}|{_AUTOMATON_KIND[0]}"]


def ranked_sources(sg, k):
    """k highest out-degree vertices, ties to the lowest id (multigpu.ranked_sources)."""
    from paper_2412_10287_b200.multigpu import ranked_sources as rs

    return rs(sg.out_degree(), k)


def read_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def per_level_roofline(st0, level_ns, x, pairs, nstates, nv, peak):
    """SURVEY §8(d) bytes per level -- 4 E_L + 8 X_L + 8 |F_L| + 2 ceil(|Q||V|/8),
    E_L the push-model edges out of F_L (counted by the untimed count_te run,
    pull levels included), X_L = |F_L| x (X / |P|) -- over the level's median
    device time (decision to decision, from the kernel's own stamps)."""
    iters = int(st0.iterations)
    out = []
    for L in range(min(iters, 63)):
        ts = [(ln[L + 1] - ln[L]) / 1e3 for ln in level_ns if len(ln) > L + 1 and ln[L + 1] > ln[L]]
        if not ts:
            break
        t_us = statistics.median(ts)
        f = int(st0.level_new[L])
        e = int(st0.level_edges[L])
        b = 4 * max(e, 0) + 8 * (f * x / max(pairs, 1)) + 8 * f + 2 * math.ceil(nstates * nv / 8)
        gbs = b / (t_us * 1e-6) / 1e9 if t_us > 0 else 0.0
        out.append({"level": L, "dir": "pull" if st0.level_dir[L] else "push", "frontier": f, "edges": e,
                    "bytes": int(b), "us": round(t_us, 2), "gbs": round(gbs, 1), "frac": round(gbs / peak, 4)})
    return out


def ncu_traffic(config):
    """DRAM bytes per launch of the step kernel from the committed ncu --set
    full capture (profiles/ncu_dram_bytes.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_dram_bytes.json")) as fh:
            return float(json.load(fh)[config]["dram_bytes_per_launch"])
    except Exception:
        return None


class ClockSampler:
    """SM clocks / throttle reasons sampled during the timed region (NVML every
    millisecond; nvidia-smi as the fallback)."""

    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap", "utilization.gpu"]

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _poll_nvml(self):
        """NVML (pynvml) polling every millisecond; False if NVML is unusable."""
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(int(self.index))
            smax = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            get_reasons = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
        except Exception:
            return False
        bits = [0x8, 0x40, 0x20, 0x4]  # hw_slowdown, hw_thermal, sw_thermal, sw_power_cap
        while not self._stop.is_set():
            try:
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                r = get_reasons(h)
                util = pynvml.nvmlDeviceGetUtilizationRates(h).gpu
                self.samples.append([str(sm), str(smax)] + ["Active" if r & b else "Not Active" for b in bits]
                                    + [str(util)])
            except Exception:
                pass
            self._stop.wait(0.001)
        return True

    def _poll(self):
        if self._poll_nvml():
            return
        cmd = ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + ",".join(self.FIELDS),
               "--format=csv,noheader,nounits"]
        while not self._stop.is_set():
            try:
                out = subprocess.run(cmd, capture_output=True, text=True, timeout=5).stdout.strip()
                parts = [p.strip() for p in out.split(",")]
                if len(parts) == len(self.FIELDS):
                    self.samples.append(parts)
            except Exception:
                pass
            self._stop.wait(0.05)

    def start(self):
        self._t = threading.Thread(target=self._poll, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        if not self.samples:
            self._stop.clear()
            self._stop.set()
        return self.summary()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        busy = [float(s[0]) for s in self.samples
                if s[0].replace(".", "").isdigit() and s[6].isdigit() and int(s[6]) > 0]
        reasons = set()
        for s in self.samples:
            for name, v in zip(["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                                "sw_power_cap"], s[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {
            "sm_mhz": statistics.median(busy or sm) if (busy or sm) else None,
            "sm_max_mhz": float(self.samples[0][1]) if self.samples[0][1].replace(".", "").isdigit() else None,
            "reasons": sorted(reasons),
            "samples": len(self.samples),
            "samples_busy": len(busy),
        }


def algorithmic_bytes(te, x, pairs, levels, nstates, nv):
    """4*TE + 8*X + 8*|P| + 2*L*ceil(R*|V|/8)."""
    return 4 * te + 8 * x + 8 * pairs + 2 * levels * math.ceil(nstates * nv / 8)


def workload_config(args, sg, sources, world):
    """The `config` dict both arms print (identical keys and values)."""
    return {
        "workload": WORKLOAD, "vertices": sg.nv, "edges": sg.ne, "query": QUERY,
        "sources": sources, "source_rule": SOURCE_RULE[args.config],
        "l2": "flushed before every query (256 MiB write, outside the query events)",
        "parallelism": (f"{world} GPUs, independent queries (each rank its own {len(sources)} sources)"
                        if world > 1 else "1 GPU"),
    }


def bench_sources(sg, config, world, per_rank):
    """BASELINE's source rule for the config; rank r of a weak-scaling run
    takes its own `per_rank` draws (rank 0's are the same at every N)."""
    from paper_2412_10287_b200 import datagen

    if datagen.CONFIGS[config]["sources"] in ("zero", "max_out_degree"):
        return ranked_sources(sg, world) if world > 1 else datagen.pick_sources(sg, config)
    return datagen.pick_sources(sg, config, count=per_rank * world)


def oracle_setup(sg, nj):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import OracleGraph, OracleQuery

    og = OracleGraph(sg.nv, sg.nl, sg.src, sg.dst, sg.lab)
    oq = OracleQuery(nj, sg.nl)
    oq.prepare(og)
    return og, oq


def cpu_baseline(og, oq, sources, te_by_source, seconds, engine_reach):
    """The reference algorithm's C restatement (engine.py's hybrid loop), one
    thread, a bounded sample: the bench's sources in order, cycled until
    `seconds` of CPU work (at least one pass).  Every source's answer is
    compared with the engine's (`parity_with_engine`)."""
    from oracle import oracle_port

    runs, total, te, parity = 0, 0.0, 0, True
    while total < seconds or runs < len(sources):
        s = sources[runs % len(sources)]
        reach, st = oracle_port(og, oq, s, "hybrid", 100.0)
        total += st["seconds"]
        te += te_by_source[s]
        if runs < len(sources):
            parity &= bool((reach == engine_reach[s]).all())
        runs += 1
    return {
        "value": te / total / 1e9,
        "unit": UNIT,
        "cores": 1,
        "kind": "port",
        "sample": (f"{args_config()} {QUERY}: {runs} sequential evaluations cycling over the bench's "
                   f"{len(sources)} sources ({total:.1f} s) by oracle/rpq_oracle.c oracle_port "
                   f"(engine.py hybrid loop, sorted-key sparse Boolean ops), 1 thread"),
        "ms_per_query": 1e3 * total / runs,
        "parity_with_engine": parity,
        "parity_sources": len(sources),
    }


_CONFIG_NAME = [CONFIG]


def args_config():
    return _CONFIG_NAME[0]


def select_workload(config):
    global QUERY, WORKLOAD
    QUERY, WORKLOAD = WORKLOADS[config]
    _CONFIG_NAME[0] = config


def run_reference(args, rank, world):
    """The reference algorithm on the host cores: each step evaluates every
    bench source concurrently, replicated to fill all host threads."""
    if rank != 0:
        return None
    from concurrent.futures import ThreadPoolExecutor

    from oracle import oracle_bfs, oracle_port
    from paper_2412_10287_b200 import datagen

    select_workload(args.config)
    sg = datagen.generate(args.config)
    nj = load_automaton(args.config, QUERY)
    all_sources = bench_sources(sg, args.config, world, args.sources or 8)
    sources = all_sources[: len(all_sources) // world]  # rank 0's share: the host runs one rank's work
    og, oq = oracle_setup(sg, nj)
    te = {s: oracle_bfs(og, oq, s)[1]["te"] for s in sources}
    threads = os.cpu_count() or 1
    reps = max(1, threads // len(sources))
    jobs = [s for _ in range(reps) for s in sources]
    pool = ThreadPoolExecutor(max_workers=min(threads, len(jobs)))

    def step():
        t = time.perf_counter()
        list(pool.map(lambda s: oracle_port(og, oq, s, "hybrid", 100.0), jobs))
        return time.perf_counter() - t

    for _ in range(args.warmup):
        step()
    times = [step() for _ in range(args.steps)]
    total = sum(times)
    te_step = sum(te[s] for s in jobs)
    value = te_step * args.steps / total / 1e9
    return {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": workload_config(args, sg, all_sources, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": min(threads, len(jobs)), "kind": "port",
                         "sample": (f"each step: {len(jobs)} concurrent evaluations ({reps} x the "
                                    f"{len(sources)} bench sources, one per host thread) of {QUERY} by "
                                    "oracle/rpq_oracle.c oracle_port (engine.py hybrid loop)"),
                         "te_per_step": te_step},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def apply_tuning(P, pq, args):
    pq.set_tuning(args.emit_mode, args.emit_inline_max)
    lib = P._lib.engine()
    for key, val, name in ((P._lib.TUNE_FLAGS, args.flags, "flags"), (P._lib.TUNE_DEFER, args.defer, "defer"),
                           (P._lib.TUNE_ZERO_COPY, args.zero_copy, "zero_copy")):
        if val is not None:
            P.engine.raise_for_status(lib.rpq_query_set_tuning(pq.q, key, float(val)), name)


def run_engine(args, rank, world, local_rank):
    import numpy as np
    import torch

    import paper_2412_10287_b200 as P
    from paper_2412_10287_b200 import datagen

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    select_workload(args.config)
    sg = datagen.generate(args.config)
    if args.reorder:
        deg = np.bincount(sg.src, minlength=sg.nv) + np.bincount(sg.dst, minlength=sg.nv)
        newid = np.empty(sg.nv, dtype=np.int32)
        newid[np.argsort(-deg, kind="stable")] = np.arange(sg.nv, dtype=np.int32)
        sg.src, sg.dst = newid[sg.src], newid[sg.dst]
        del deg, newid
    g = sg.labeled_graph()
    nj = load_automaton(args.config, QUERY)
    n = P.Automaton.from_json(nj)
    all_sources = bench_sources(sg, args.config, world, args.sources or 8)
    if args.source is not None:
        all_sources = [args.source] * world
    per = len(all_sources) // world
    sources = all_sources[rank * per:(rank + 1) * per]
    pq = P.PreparedQuery(g, n, device=local_rank)
    # a dedicated (non-default) stream: the engine and the timing events share it
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    handle = stream.cuda_stream
    assert handle, "need a real stream handle"
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    apply_tuning(P, pq, args)

    # one untimed run per source for its work counts (exact TE, |P|, levels)
    alpha = args.alpha if args.alpha is not None else P.EngineOptions().alpha
    outdeg_q = np.bincount(pq.table.t_src, minlength=pq.table.nstates)
    work = {}
    for s in sources:
        pq.set_options(direction=args.direction, count_te=True, alpha=alpha)
        pq.launch(s, -1.0, handle)
        st0 = pq.wait()
        x = int((pq.visited_counts() * outdeg_q).sum())
        te, pairs, iters = int(st0.te), int(st0.visited_pairs), int(st0.iterations)
        work[s] = {"st0": st0, "te": te, "x": x, "pairs": pairs, "iters": iters,
                   "bytes": algorithmic_bytes(te, x, pairs, iters, pq.table.nstates, sg.nv),
                   "reach": pq.reach()}
    pq.set_options(direction=args.direction, count_te=False, alpha=alpha)

    sampler = None
    if not args.profile:
        phys = os.environ.get("CUDA_VISIBLE_DEVICES", str(local_rank)).split(",")[local_rank]
        sampler = ClockSampler(phys)
        sampler.start()

    for i in range(args.warmup):
        for s in sources:
            flush.fill_(i & 0xFF)
            pq.launch(s, -1.0, handle)
            pq.wait()

    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in sources]
          for _ in range(args.steps)]
    launches = 0
    level_ns = {s: [] for s in sources}  # per timed query: the kernel's own level stamps
    for k in range(args.steps):
        for j, s in enumerate(sources):
            if not args.no_flush:
                flush.fill_((k + j) & 0xFF)  # > L2: evicts the graph between queries (outside the events)
            ev[k][j][0].record(stream)
            pq.launch(s, -1.0, handle)
            launches += 1
            ev[k][j][1].record(stream)
            st = pq.wait()
            w = work[s]
            assert st.visited_pairs == w["pairs"] and st.iterations == w["iters"]
            level_ns[s].append(list(st.level_ns[: min(w["iters"] + 1, 64)]))
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    q_ms = {s: [ev[k][j][0].elapsed_time(ev[k][j][1]) for k in range(args.steps)] for j, s in enumerate(sources)}
    total_ms = sum(sum(v) for v in q_ms.values())
    te_step = sum(work[s]["te"] for s in sources)
    b_step = sum(work[s]["bytes"] for s in sources)

    # e2e through the public API: automaton H2D + kernel + answer D2H per call
    e2e_s, set_ms, e2e_dev_ms, d2h_answer, e2e_host_us, view_us = [], [], [], {}, [], []
    host_answered = set()
    nwords = (sg.nv + 31) // 32
    if not args.profile:
        opts = P.EngineOptions(timeout=math.inf, direction=args.direction, alpha=alpha)
        for _ in range(args.warmup):  # untimed, like the device leg (first call creates the query)
            for s in sources:
                P.eval_ssr(g, n, s, opts)
        for k in range(args.steps):
            t_step = 0.0
            for j, s in enumerate(sources):
                flush.fill_((k + j) & 0xFF)
                torch.cuda.synchronize()
                t = time.perf_counter()
                res = P.eval_ssr(g, n, s, opts)
                dt = time.perf_counter() - t
                t_step += dt
                e2e_dev_ms.append(P.engine._thread_stats().device_ms)  # this call's device time
                e2e_host_us.append(1e6 * dt - 1e3 * e2e_dev_ms[-1])
                if k == 0 and P.engine._thread_stats().grid == 0:
                    host_answered.add(s)  # no seed edge: answered without a launch
                assert res.iterations == work[s]["iters"]
                if s not in d2h_answer:  # bytes the answer took over PCIe: bitmap or (word, bits) pairs
                    nz = int(np.count_nonzero(res.bits))
                    d2h_answer[s] = 8 * nz if 2 * nz < nwords else 4 * nwords
                if k == 0:
                    assert np.array_equal(res.reach, work[s]["reach"])
                del res
            e2e_s.append(t_step)
        # after the timed calls (the millions of Python ints of a reference-style
        # set would otherwise leave garbage-collector work inside them): the
        # cost of the reference's result type, set[int], and of the lazy view
        for s in sources:
            res = P.eval_ssr(g, n, s, opts)
            t = time.perf_counter()
            view = res.answer_set
            assert len(view) == int(work[s]["st0"].reach_count)
            view_us.append(1e6 * (time.perf_counter() - t))
            t = time.perf_counter()
            _ = res.reachable
            set_ms.append(1e3 * (time.perf_counter() - t))
            del res, view, _
    clocks = sampler.stop() if sampler else None

    h2d, d2h_ctl = pq.io_bytes()
    from paper_2412_10287_b200.multigpu import reduce_timing

    # max over ranks of the device time, sum over ranks of the product edges
    total_max_ms, units = reduce_timing(total_ms, te_step * args.steps, dev)
    peak, peak_src = read_peaks()
    heavy = max(sources, key=lambda s: work[s]["te"])
    hw = work[heavy]
    per_level = per_level_roofline(hw["st0"], level_ns[heavy], hw["x"], hw["pairs"], pq.table.nstates,
                                   sg.nv, peak)
    e2e_max_s, _ = reduce_timing(sum(e2e_s) if e2e_s else 0.0, 0, dev)
    cfg = workload_config(args, sg, all_sources, world)
    pq.close()
    if rank != 0:
        return None

    value = units / (total_max_ms / 1e3) / 1e9
    kernel_s = total_ms / args.steps / 1e3  # one step = every source once
    achieved = b_step / kernel_s / 1e9
    nq = len(sources)
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_max_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic",
        "config": cfg,
        "per_query": {
            "sources": sources,
            "latency_ms_median": {str(s): statistics.median(q_ms[s]) for s in sources},
            "latency_ms_median_all": statistics.median([t for s in sources for t in q_ms[s]]),
            "te": {str(s): work[s]["te"] for s in sources},
            "iterations": {str(s): work[s]["iters"] for s in sources},
            "reach": {str(s): int(work[s]["st0"].reach_count) for s in sources},
            "heaviest_source": heavy,
            "heaviest": {
                "latency_ms_median": statistics.median(q_ms[heavy]), "te": hw["te"], "x": hw["x"],
                "visited_pairs": hw["pairs"], "iterations": hw["iters"],
                "level_new": list(hw["st0"].level_new[: hw["iters"] + 1]),
                "level_edges": list(hw["st0"].level_edges[: hw["iters"] + 1]),
                "level_dir": ["pull" if d else "push" for d in hw["st0"].level_dir[: hw["iters"]]],
            },
            "direction_policy": args.direction,
        },
        "roofline": {
            "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": ncu_traffic(args.config),
            "kernel": "rpq_ssr_kernel (persistent, one launch per query)",
            "algorithmic_bytes_per_step": b_step, "queries_per_step": nq,
            "algorithmic_bytes_per_launch": b_step / nq, "peak_source": peak_src,
            "note": ("SURVEY.md §8(d) algorithmic bytes summed over the step's queries / the step's summed "
                     "query times; traffic = ncu dram bytes of one launch of the heaviest source"),
            "per_level_heaviest_source": per_level,
            # the frontier step with the most edges (north_star's "frontier step" figure)
            "densest_level_frac": max(per_level, key=lambda lv: lv["edges"])["frac"] if per_level else None,
        },
        "gpu_launches": launches,
        "clocks": clocks,
    }
    if e2e_s:
        nlaunched = nq - len(host_answered)
        out["e2e"] = {"value": units / e2e_max_s / 1e9, "unit": UNIT,
                      "h2d_bytes_per_step": nlaunched * (h2d + 4),
                      "d2h_bytes_per_step": nlaunched * d2h_ctl + sum(d2h_answer.get(s, 0) for s in sources),
                      "host_answered_queries_per_step": len(host_answered),
                      "latency_ms_median_per_query": 1e3 * statistics.median(e2e_s) / nq,
                      "device_ms_per_query": statistics.mean(e2e_dev_ms) if e2e_dev_ms else None,
                      "host_us_per_query": {"median": statistics.median(e2e_host_us),
                                            "mean": statistics.mean(e2e_host_us)} if e2e_host_us else None,
                      "reachable_set_ms_per_query": statistics.mean(set_ms) if set_ms else None,
                      "answer_set_view_us_per_query": statistics.mean(view_us) if view_us else None,
                      "note": ("eval_ssr per source with host buffers: automaton tables H2D, the answer D2H as "
                               "the bitmap or, when sparse, (word, bits) pairs; device_ms = the calls' own "
                               "CUDA-event time; reachable_set_ms = building the reference's set[int] from the "
                               "answer, not in value; host_answered_queries_per_step = sources none of whose "
                               "seed rows has an edge (empty first step, engine.py:154-160): eval_ssr answers "
                               "them from the host copy of the row bitmaps without a launch -- `value` still "
                               "times a kernel for every source")}
    if world == 1 and not args.no_cpu_baseline and not args.profile:
        og, oq = oracle_setup(sg, nj)
        out["cpu_baseline"] = cpu_baseline(og, oq, sources, {s: work[s]["te"] for s in sources},
                                           args.cpu_seconds, {s: work[s]["reach"] for s in sources})
    return out


def _timed_flush(flush, i):
    flush.fill_(i & 0xFF)  # > L2: evicts the graph between queries (outside the events)


def run_partitioned(args, rank, world, local_rank):
    """One query at a time over all ranks, vertex-partitioned 1-D (SURVEY.md
    §8(e) regime 2): every rank runs the step kernel on its owned targets and
    the owned slices of the next frontier are allgathered (NCCL) per level.
    Strong scaling: every rank evaluates the same sources; value = sum of TE /
    the max over ranks of the device-timed query time."""
    import numpy as np
    import torch

    import paper_2412_10287_b200 as P
    from paper_2412_10287_b200 import datagen
    from paper_2412_10287_b200.multigpu import reduce_timing
    from paper_2412_10287_b200.partition import partitioned_query

    dev = torch.device("cuda", local_rank)
    select_workload(args.config)
    sg = datagen.generate(args.config)
    g = sg.labeled_graph()
    nj = load_automaton(args.config, QUERY)
    n = P.Automaton.from_json(nj)
    sources = bench_sources(sg, args.config, 1, args.sources or 8)
    if args.source is not None:
        sources = [args.source]
    # exact work per source (TE, levels) from the fused kernel on the full graph
    work = {}
    with P.PreparedQuery(g, n, device=local_rank) as fq:
        fq.set_options(count_te=True)
        for s in sources:
            fq.launch(s, -1.0, None)
            st = fq.wait()
            work[s] = {"te": int(st.te), "iters": int(st.iterations), "reach": fq.reach()}
    pq = partitioned_query(g, n)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    for i in range(args.warmup):
        for s in sources:
            words, its, _ = pq.run(s)
            assert its == work[s]["iters"], (s, its, work[s]["iters"])
            if i == 0:
                got = np.unpackbits(words.view(np.uint8), bitorder="little")[: sg.nv]
                assert np.array_equal(got, work[s]["reach"]), s
    sampler = None
    if not args.profile:
        phys = os.environ.get("CUDA_VISIBLE_DEVICES", str(local_rank)).split(",")[local_rank]
        sampler = ClockSampler(phys)
        sampler.start()
    torch.distributed.barrier()
    torch.cuda.synchronize()
    cur = torch.cuda.current_stream(dev)
    q_ms = {s: [] for s in sources}
    for k in range(args.steps):
        for j, s in enumerate(sources):
            _timed_flush(flush, k + j)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(cur)
            _, its, _ = pq.run(s)
            e1.record(cur)
            e1.synchronize()
            q_ms[s].append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    torch.distributed.barrier()
    clocks = sampler.stop() if sampler else None
    total_ms = sum(sum(v) for v in q_ms.values())
    te_step = sum(work[s]["te"] for s in sources)
    total_max_ms, _ = reduce_timing(total_ms, 0, dev)
    # per-level wall timings of the heaviest source (one profiled run)
    heavy = max(sources, key=lambda s: work[s]["te"])
    _, _, prof = pq.run(heavy, profile=True)
    # e2e: the public call (answer bitmap gathered to the host)
    e2e = []
    if not args.profile:
        for k in range(args.steps):
            t_step = 0.0
            for j, s in enumerate(sources):
                _timed_flush(flush, k + j)
                torch.cuda.synchronize()
                torch.distributed.barrier()
                t = time.perf_counter()
                res = P.partition.eval_ssr_partitioned(g, n, s, P.EngineOptions(timeout=math.inf))
                t_step += time.perf_counter() - t
                assert res.iterations == work[s]["iters"]
            e2e.append(t_step)
    e2e_max, _ = reduce_timing(sum(e2e) if e2e else 0.0, 0, dev)
    if rank != 0:
        return None
    value = te_step * args.steps / (total_max_ms / 1e3) / 1e9
    ranges = pq.ranges
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_max_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": {**workload_config(args, sg, sources, 1),
                   "parallelism": f"{world} GPU(s), one query vertex-partitioned 1-D over all ranks "
                                  f"(NCCL allgather of the owned frontier slices per level)"},
        "mode": "partitioned",
        "per_query": {
            "latency_ms_median": {str(s): statistics.median(q_ms[s]) for s in sources},
            "te": {str(s): work[s]["te"] for s in sources},
            "iterations": {str(s): work[s]["iters"] for s in sources},
            "heaviest_source": heavy,
            "heaviest_level_wall_us": prof["levels_wall_us"],
            "heaviest_step_ms": prof["step_ms"],
        },
        "partition": {"ranks": world, "word_ranges": [list(r) for r in ranges],
                      "exchange_bytes_per_level": int(pq.table.nstates * max(w1 - w0 for w0, w1 in ranges) * 4
                                                      * world)},
        "gpu_launches": None,
        "clocks": clocks,
    }
    if e2e:
        out["e2e"] = {"value": te_step * args.steps / e2e_max / 1e9, "unit": UNIT,
                      "h2d_bytes_per_step": 0, "d2h_bytes_per_step": len(sources) * ((sg.nv + 31) // 32) * 4,
                      "note": "eval_ssr_partitioned per source; the answer bitmap gathered and read back"}
    return out


def run_batch_mode(args, rank, world, local_rank):
    """Multi-source throughput: the config's source set (cfg5: 1,024 uniform
    sources) sharded over ranks, 64 sources per launch of the bit-sliced batch
    kernel; value = sum of TE over all sources / max over ranks of the
    device time.  Weak scaling in the sources per rank."""
    import torch

    import paper_2412_10287_b200 as P
    from paper_2412_10287_b200 import datagen
    from paper_2412_10287_b200.multigpu import reduce_timing

    dev = torch.device("cuda", local_rank)
    select_workload(args.config)
    sg = datagen.generate(args.config)
    g = sg.labeled_graph()
    nj = load_automaton(args.config, QUERY)
    n = P.Automaton.from_json(nj)
    total = args.sources or datagen.CONFIGS[args.config].get("nsources", 32)
    all_sources = datagen.pick_sources(sg, args.config, count=total * world)
    per = len(all_sources) // world
    sources = all_sources[rank * per:(rank + 1) * per]
    pq = P.PreparedQuery(g, n, device=local_rank)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    batches = [sources[b:b + P._lib.BATCH] for b in range(0, len(sources), P._lib.BATCH)]
    te = 0
    for b in batches:
        pq.launch_batch(b, -1.0, stream.cuda_stream)
        te += int(pq.wait_batch().te)
    for _ in range(args.warmup):
        for b in batches:
            pq.launch_batch(b, -1.0, stream.cuda_stream)
            pq.wait_batch()
    sampler = None
    if not args.profile:
        phys = os.environ.get("CUDA_VISIBLE_DEVICES", str(local_rank)).split(",")[local_rank]
        sampler = ClockSampler(phys)
        sampler.start()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    ms = 0.0
    launches = 0
    for k in range(args.steps):
        for i, b in enumerate(batches):
            _timed_flush(flush, k + i)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            pq.launch_batch(b, -1.0, stream.cuda_stream)
            e1.record(stream)
            st = pq.wait_batch()
            launches += 1
            ms += e0.elapsed_time(e1)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    clocks = sampler.stop() if sampler else None
    ms_max, te_all = reduce_timing(ms, te * args.steps, dev)
    pq.close()
    if rank != 0:
        return None
    return {
        "metric": METRIC, "value": te_all / (ms_max / 1e3) / 1e9, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic",
        "config": {**workload_config(args, sg, all_sources[:4] + ["..."], world),
                   "sources_total": len(all_sources), "sources_per_rank": per,
                   "parallelism": f"{world} GPU(s), sources sharded over ranks, 64 per batch-kernel launch"},
        "mode": "batch", "gpu_launches": launches, "clocks": clocks,
    }


def main():
    args = parse_args()
    _AUTOMATON_KIND[0] = args.automaton
    # stdout carries exactly one JSON line: anything else that writes to fd 1
    # (NCCL's version banner, library chatter) goes to stderr
    sys.stdout.flush()
    json_out = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus if args.gpus == 1 else 1)))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        out = run_reference(args, rank, world)
    else:
        dist_needed = world > 1 or args.mode == "partitioned"
        if dist_needed:
            import torch

            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29511")
            os.environ.setdefault("RANK", str(rank))
            os.environ.setdefault("WORLD_SIZE", str(world))
            torch.cuda.set_device(local_rank)
            torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        if args.mode == "partitioned":
            out = run_partitioned(args, rank, world, local_rank)
        elif args.mode == "batch":
            out = run_batch_mode(args, rank, world, local_rank)
        else:
            out = run_engine(args, rank, world, local_rank)
        if dist_needed:
            import torch

            torch.distributed.destroy_process_group()
    if out is not None:
        json_out.write(json.dumps(out) + "\n")
        json_out.flush()


if __name__ == "__main__":
    main()
