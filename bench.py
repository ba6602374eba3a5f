#!/usr/bin/env python
"""Benchmark: 2-RPQ product edges traversed per second (GTEPS) and per-query
latency on the BASELINE.json headline configuration (configs[1] = cfg2):

  R-MAT scale 20 (1,048,576 vertices), edge factor 16, (0.57, 0.19, 0.19, 0.05),
  self-loops and duplicates removed, 16 Zipf(1.0) labels; two-way query
  a ^b* c (the reference compiler's minimal 3-state DFA); source = the vertex
  with the highest out-degree.  Synthetic, seeded (paper_2412_10287_b200/datagen.py).

A step is one single-source query evaluation (seed -> answer vector ready on
the device).  `value` is device-timed with CUDA events around each step on
the launching stream (inputs resident in HBM, L2 flushed between steps);
`e2e` is the same metric through the public API `eval_ssr` with the automaton
sent host->device every call and the uint8 answer read back to the host.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl engine|reference]

With N > 1 (torchrun, one rank per GPU) every rank evaluates its own
independent query -- rank r starts from the r-th highest out-degree vertex --
with no data-path collective (weak scaling over independent queries).
`--impl reference` times the reference algorithm's CPU restatement
(oracle/rpq_oracle.c oracle_port, the hybrid loop of engine.py:197-232) on all
host cores, one independent query per thread; rank 0 only.
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

METRIC = "2-RPQ edges traversed/sec (GTEPS)"
UNIT = "GTEPS"
CONFIG = "cfg2"
QUERY = "a ^b* c"
WORKLOADS = {
    "cfg1": ("a b*", "cfg1: Erdos-Renyi 10,000 V / 100,000 E, 4 uniform labels, query a b* "
                     "(2-state min DFA), source 0"),
    "cfg2": ("a ^b* c", "cfg2: R-MAT scale 20 (1,048,576 V), edge factor 16, abc=(0.57,0.19,0.19), "
                        "16 Zipf(1.0) labels, query a ^b* c (3-state min DFA), source = max out-degree"),
    "cfg3": ("^a (b|c)* d", "cfg3: R-MAT scale 24 (16,777,216 V), edge factor 16, 64 Zipf(1.0) labels, "
                            "query ^a (b|c)* d (3-state min DFA), source = max out-degree"),
    "cfg4": ("(a|b|c|d)*", "cfg4: Chung-Lu 90M V / 1.2B raw edges (exponent 2.1), 2,000 Zipf(1.1) labels, "
                           "query (a|b|c|d)* (1-state min DFA), source = max out-degree"),
    "cfg5": ("(a1 a2*) (a3 a4*) (a5 a6*) (a7 a8*) (a9 a10*) (a11 a12*) (a13 a14*) (a15 a16*)",
             "cfg5: R-MAT scale 22, 32 Zipf(1.0) labels, 8-group chain query (9-state min DFA), "
             "source = max out-degree"),
}
WORKLOAD = WORKLOADS[CONFIG][1]
L2_FLUSH_BYTES = 256 << 20


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["engine", "reference"], default="engine")
    ap.add_argument("--config", default=CONFIG)
    ap.add_argument("--no-cpu-baseline", action="store_true")
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
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-flush", action="store_true", help="keep L2 warm between steps (diagnostic)")
    ap.add_argument("--profile", action="store_true",
                    help="short run for ncu: no e2e leg, no CPU baseline, no clocks")
    return ap.parse_args()


def load_automaton(config, query):
    with open(os.path.join(ROOT, "paper_2412_10287_b200", "data", "config_automata.json")) as fh:
        return json.load(fh)[config][f"{query}|min"]


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


def cpu_baseline(sg, nj, source, seconds, engine_reach):
    """The reference algorithm's C restatement, one thread, bounded sample."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import OracleGraph, OracleQuery, oracle_port

    og = OracleGraph(sg.nv, sg.nl, sg.src, sg.dst, sg.lab)
    oq = OracleQuery(nj, sg.nl)
    oq.prepare(og)
    runs, total, te = 0, 0.0, None
    reach = None
    while total < seconds or runs == 0:
        reach, st = oracle_port(og, oq, source, "hybrid", 100.0)
        total += st["seconds"]
        runs += 1
    from oracle import oracle_bfs

    _, bst = oracle_bfs(og, oq, source)
    te = bst["te"]
    return {
        "value": te * runs / total / 1e9,
        "unit": UNIT,
        "cores": 1,
        "kind": "port",
        "sample": (f"{CONFIG} {QUERY} from source {source}, {runs} sequential evaluations "
                   f"({total:.1f} s) by oracle/rpq_oracle.c oracle_port (engine.py hybrid loop, "
                   f"sorted-key sparse Boolean ops), 1 thread"),
        "ms_per_query": 1e3 * total / runs,
        "parity_with_engine": bool((reach == engine_reach).all()),
    }


def run_reference(args, rank, world):
    if rank != 0:
        return None
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from concurrent.futures import ThreadPoolExecutor

    from oracle import OracleGraph, OracleQuery, oracle_bfs, oracle_port
    from paper_2412_10287_b200 import datagen

    global QUERY, WORKLOAD
    QUERY, WORKLOAD = WORKLOADS[args.config]
    sg = datagen.generate(args.config)
    nj = load_automaton(args.config, QUERY)
    source = ranked_sources(sg, 1)[0]
    og = OracleGraph(sg.nv, sg.nl, sg.src, sg.dst, sg.lab)
    oq = OracleQuery(nj, sg.nl)
    oq.prepare(og)
    _, bst = oracle_bfs(og, oq, source)
    te = bst["te"]
    threads = os.cpu_count() or 1
    pool = ThreadPoolExecutor(max_workers=threads)

    def step():
        t = time.perf_counter()
        list(pool.map(lambda _: oracle_port(og, oq, source, "hybrid", 100.0), range(threads)))
        return time.perf_counter() - t

    for _ in range(args.warmup):
        step()
    times = [step() for _ in range(args.steps)]
    total = sum(times)
    value = threads * te * args.steps / total / 1e9
    return {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "vertices": sg.nv, "edges": sg.ne, "query": QUERY,
                   "source": source, "te_per_query": te},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": (f"each step: {threads} concurrent evaluations of {QUERY} from "
                                    f"source {source} (one per host thread) by "
                                    "oracle/rpq_oracle.c oracle_port (hybrid loop)")},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def run_engine(args, rank, world, local_rank):
    import numpy as np
    import torch

    import paper_2412_10287_b200 as P
    from paper_2412_10287_b200 import datagen

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    global QUERY, WORKLOAD
    QUERY, WORKLOAD = WORKLOADS[args.config]
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
    source = ranked_sources(sg, world)[rank]
    pq = P.PreparedQuery(g, n, device=local_rank)
    # a dedicated (non-default) stream: the engine and the timing events share it
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    handle = stream.cuda_stream
    assert handle, "need a real stream handle"
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)

    pq.set_tuning(args.emit_mode, args.emit_inline_max)
    if args.flags is not None:
        P.engine.raise_for_status(P._lib.engine().rpq_query_set_tuning(pq.q, P._lib.TUNE_FLAGS, float(args.flags)), "flags")
    if args.defer is not None:
        P.engine.raise_for_status(P._lib.engine().rpq_query_set_tuning(pq.q, P._lib.TUNE_DEFER, float(args.defer)), "defer")
    if args.zero_copy is not None:
        P.engine.raise_for_status(P._lib.engine().rpq_query_set_tuning(pq.q, P._lib.TUNE_ZERO_COPY, float(args.zero_copy)),
                                  "zero_copy")
    # one untimed run for the work counts (exact TE, |P|, levels) of this query
    alpha = args.alpha if args.alpha is not None else P.EngineOptions().alpha
    pq.set_options(direction=args.direction, count_te=True, alpha=alpha)
    pq.launch(source, -1.0, handle)
    st0 = pq.wait()
    pq.set_options(direction=args.direction, count_te=False, alpha=alpha)
    per_state = pq.visited_counts()
    outdeg_q = np.bincount(pq.table.t_src, minlength=pq.table.nstates)
    x = int((per_state * outdeg_q).sum())
    te, pairs, iters = int(st0.te), int(st0.visited_pairs), int(st0.iterations)
    b_alg = algorithmic_bytes(te, x, pairs, iters, pq.table.nstates, sg.nv)
    engine_reach = pq.reach()

    sampler = None
    if not args.profile:
        phys = os.environ.get("CUDA_VISIBLE_DEVICES", str(local_rank)).split(",")[local_rank]
        sampler = ClockSampler(phys)
        sampler.start()

    for i in range(args.warmup):
        flush.fill_(i & 0xFF)
        pq.launch(source, -1.0, handle)
        pq.wait()

    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    launches = 0
    level_ns = []  # per timed step: the kernel's own level stamps
    for k in range(args.steps):
        if not args.no_flush:
            flush.fill_(k & 0xFF)  # > L2: evicts the graph between steps (outside the events)
        ev[k][0].record(stream)
        pq.launch(source, -1.0, handle)
        launches += 1
        ev[k][1].record(stream)
        st = pq.wait()
        assert st.visited_pairs == pairs and st.iterations == iters
        level_ns.append(list(st.level_ns[: min(iters + 1, 64)]))
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = sum(step_ms)

    # e2e through the public API: automaton H2D + kernel + answer D2H per call
    e2e_s = []
    if not args.profile:
        opts = P.EngineOptions(timeout=math.inf, direction=args.direction, alpha=alpha)
        for _ in range(args.warmup):  # untimed, like the device leg (first call creates the query)
            P.eval_ssr(g, n, source, opts)
        for k in range(args.steps):
            flush.fill_(k & 0xFF)
            torch.cuda.synchronize()
            t = time.perf_counter()
            res = P.eval_ssr(g, n, source, opts)
            e2e_s.append(time.perf_counter() - t)
            assert res.iterations == iters
        assert np.array_equal(res.reach, engine_reach)
    clocks = sampler.stop() if sampler else None

    h2d, d2h_ctl = pq.io_bytes()
    d2h = d2h_ctl + (sg.nv + 31) // 32 * 4  # eval_ssr reads back the answer bitmap
    from paper_2412_10287_b200.multigpu import reduce_timing

    # max over ranks of the device time, sum over ranks of the product edges
    total_max_ms, units = reduce_timing(total_ms, te * args.steps, dev)
    peak, peak_src = read_peaks()
    per_level = per_level_roofline(st0, level_ns, x, pairs, pq.table.nstates, sg.nv, peak)
    e2e_max_s, _ = reduce_timing(sum(e2e_s) if e2e_s else 0.0, 0, dev)
    pq.close()
    if rank != 0:
        return None

    value = units / (total_max_ms / 1e3) / 1e9
    kernel_s = total_ms / args.steps / 1e3
    achieved = b_alg / kernel_s / 1e9
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_max_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic",
        "config": {
            "workload": WORKLOAD, "vertices": sg.nv, "edges": sg.ne, "query": QUERY,
            "automaton_states": pq.table.nstates, "sources": ranked_sources(sg, world),
            "l2": "flushed between steps (256 MiB write, outside the step events)",
            "parallelism": f"{world} independent queries (1 per GPU)" if world > 1 else "1 GPU",
        },
        "per_query": {
            "latency_ms_median": statistics.median(step_ms), "latency_ms_min": min(step_ms),
            "te": te, "x": x, "visited_pairs": pairs, "iterations": iters,
            "reach": int(st0.reach_count),
            "level_new": list(st0.level_new[: iters + 1]),
            "level_edges": list(st0.level_edges[: iters + 1]),
            "level_dir": ["pull" if d else "push" for d in st0.level_dir[: iters]],
            "level_end_us": [t / 1e3 for t in st0.level_ns[: iters + 1]],
            "level_work_us": [t / 1e3 for t in st0.work_ns[: iters]],
            "level_bar_us": [t / 1e3 for t in st0.bar_ns[: iters]],
            "direction_policy": args.direction,
        },
        "roofline": {
            "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": ncu_traffic(args.config),
            "kernel": "rpq_ssr_kernel (persistent, one launch per query)",
            "algorithmic_bytes_per_launch": b_alg, "peak_source": peak_src,
            "note": "algorithmic bytes of SURVEY.md §8(d) per query / mean step time",
            "per_level": per_level,
            # the frontier step with the most edges (north_star's "frontier step" figure)
            "densest_level_frac": max(per_level, key=lambda lv: lv["edges"])["frac"] if per_level else None,
        },
        "gpu_launches": launches,
        "clocks": clocks,
    }
    if e2e_s:
        out["e2e"] = {"value": units / e2e_max_s / 1e9, "unit": UNIT,
                      "h2d_bytes_per_step": h2d + 4, "d2h_bytes_per_step": d2h,
                      "latency_ms_median": 1e3 * statistics.median(e2e_s)}
    if world == 1 and not args.no_cpu_baseline and not args.profile:
        out["cpu_baseline"] = cpu_baseline(sg, nj, source, args.cpu_seconds, engine_reach)
    return out


def main():
    args = parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus if args.gpus == 1 else 1)))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        out = run_reference(args, rank, world)
    else:
        if world > 1:
            import torch

            torch.cuda.set_device(local_rank)
            torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        out = run_engine(args, rank, world, local_rank)
        if world > 1:
            import torch

            torch.distributed.destroy_process_group()
    if out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
