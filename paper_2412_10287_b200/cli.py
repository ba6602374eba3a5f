"""Benchmark front end: the reference's ``bench`` workload runner on the
device engine.

Mirrors /root/reference/pkg/src/rpq/cli.py:
  parse_workload  cli.py:48-69   TSV ``id<TAB>mode<TAB>endpoint<TAB>pattern``, same errors
  run_entry       cli.py:83-125  automaton compiled (and reversed for sdr) outside the
                                 timer; ``repeat`` runs, the first dropped when repeat >= 2,
                                 median time; status ok / timeout / error
  run_bench       cli.py:128-140 input order kept; ``workers`` threads share the graph
  write_csv       cli.py:143-157 BENCH_HEADER = id,mode,algorithm,result_count,iterations,
                                 time_ms,status (cli.py:29)

Extended rows (``write_csv(..., extended=True)``) add the throughput columns
of SURVEY.md §5: gteps, levels, te (product edges), bytes_alg
(4 TE + 8 X + 8 |P| + 2 L ceil(|Q||V|/8)), roofline_frac (bytes_alg / time /
measured HBM peak), ngpu, cpu_ms, cpu_cores.  The engine leaves the two CPU
columns empty; bench.py fills them from its CPU baseline.

``run_batch`` is the multi-source counterpart (eval_ssr_batch's kernel, 32
sources per launch): one row per source, ``time_ms`` = its launch's time
divided by the sources in that launch.

Command line (synthetic configs of BASELINE.json, or a workload TSV over one):

    python -m paper_2412_10287_b200.cli bench --config cfg3 --sources 8 --repeat 5 [--batch] [--out rows.csv]
    python -m paper_2412_10287_b200.cli bench --config cfg1 --workload wl.tsv --automata automata.json

Patterns are compiled by the reference's own compiler when it is importable
(``rpq.query_compiler.compile``), else looked up in an automata JSON (the
format of data/config_automata.json: ``"<pattern>|min"`` -> automaton).
"""

import argparse
import csv
import json
import math
import os
import statistics
import sys
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

from . import _lib
from .automaton import Automaton, reverse
from .engine import EngineOptions, PreparedQuery, QueryTimeout, eval_ssr, eval_ssr_batch

BENCH_HEADER = ["id", "mode", "algorithm", "result_count", "iterations", "time_ms", "status"]
EXT_HEADER = BENCH_HEADER + ["gteps", "levels", "te", "bytes_alg", "roofline_frac", "ngpu", "cpu_ms",
                             "cpu_cores"]


@dataclass
class WorkloadEntry:
    id: str
    mode: str  # "ssr" | "sdr"
    endpoint: str  # external vertex id
    pattern: str


class WorkloadFormatError(ValueError):
    def __init__(self, line_no, message):
        super().__init__(f"line {line_no}: {message}")
        self.line_no = line_no


def parse_workload(stream):
    """cli.py:48-69: tab-separated id, mode, endpoint, pattern; '#' comments;
    unique ids; mode ssr or sdr."""
    entries, seen = [], set()
    for line_no, raw in enumerate(stream, start=1):
        line = raw.rstrip("\r\n")
        if not line or line.startswith("#"):
            continue
        parts = line.split("\t")
        if len(parts) != 4:
            raise WorkloadFormatError(line_no, f"expected 4 tab-separated fields, got {len(parts)}")
        e = WorkloadEntry(*parts)
        if e.mode not in ("ssr", "sdr"):
            raise WorkloadFormatError(line_no, f"mode must be ssr or sdr, got {e.mode!r}")
        if e.id in seen:
            raise WorkloadFormatError(line_no, f"duplicate id {e.id!r}")
        seen.add(e.id)
        entries.append(e)
    return entries


def vertex_of(g, endpoint):
    """Dense index of an external vertex id (graph_store.py vertex_index);
    graphs without names use the decimal index itself."""
    v = g.vertex_index(endpoint) if hasattr(g, "vertex_index") else int(endpoint)
    if not 0 <= v < g.num_vertices:
        raise IndexError(f"vertex index {v} out of range")
    return v


def read_peak_gbs(root=None):
    """Measured HBM copy bandwidth (MEASURED_PEAKS.json, driver-written), or
    the profiling guide's B200 fallback."""
    path = os.path.join(root or os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                        "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"])
    except Exception:
        return 6650.0


def work_counts(g, n, vertex, opts):
    """Exact work of one evaluation (untimed): TE, X, |P|, levels and the
    SURVEY §8(d) algorithmic bytes."""
    with PreparedQuery(g, n, device=opts.device) as pq:
        pq.set_options(direction=opts.direction, count_te=True, alpha=opts.alpha)
        pq.launch(vertex, -1.0, None)
        st = pq.wait()
        outdeg_q = np.bincount(pq.table.t_src, minlength=pq.table.nstates)
        x = int((pq.visited_counts() * outdeg_q).sum())
        nstates = pq.table.nstates
    te, pairs, levels = int(st.te), int(st.visited_pairs), int(st.iterations)
    nv = int(g.num_vertices)
    b = 4 * te + 8 * x + 8 * pairs + 2 * levels * math.ceil(nstates * nv / 8)
    return {"te": te, "x": x, "pairs": pairs, "levels": levels, "bytes_alg": b}


def _empty_row(entry, opts):
    return {"id": entry.id, "mode": entry.mode, "algorithm": opts.algorithm, "result_count": 0,
            "iterations": 0, "time_ms": 0.0, "status": "ok"}


def run_entry(g, entry, opts, repeat, *, compile_fn=None, work=False, peak_gbs=None, ngpu=1):
    """cli.py:83-125 on the device engine.  ``compile_fn(pattern)`` -> automaton
    (default: the reference compiler over g's labels), outside the timer as is
    the reversal for sdr.  With ``work`` the row also carries the extended
    columns (one extra untimed counting run)."""
    row = _empty_row(entry, opts)
    try:
        vertex = vertex_of(g, entry.endpoint)
        n = (compile_fn or automaton_compiler(labels=list(g.labels)))(entry.pattern)
        if entry.mode == "sdr":
            n = reverse(n)
        times, result = [], None
        for _ in range(max(1, repeat)):
            t0 = time.perf_counter()
            result = eval_ssr(g, n, vertex, opts)
            times.append((time.perf_counter() - t0) * 1000.0)
        if len(times) >= 2:
            times = times[1:]
        row["result_count"] = int(result.reach.sum())
        row["iterations"] = result.iterations
        row["time_ms"] = statistics.median(times)
        if work:
            w = work_counts(g, n, vertex, opts)
            row.update(_ext_columns(w, row["time_ms"], peak_gbs or read_peak_gbs(), ngpu))
    except QueryTimeout:
        row["status"] = "timeout"
        row["time_ms"] = opts.timeout * 1000.0
    except (KeyError, ValueError, IndexError):
        row["status"] = "error"
    return row


def _ext_columns(w, time_ms, peak_gbs, ngpu):
    s = time_ms / 1e3
    return {"gteps": w["te"] / s / 1e9 if s > 0 else 0.0, "levels": w["levels"], "te": w["te"],
            "bytes_alg": w["bytes_alg"], "roofline_frac": w["bytes_alg"] / s / 1e9 / peak_gbs if s > 0 else 0.0,
            "ngpu": ngpu, "cpu_ms": "", "cpu_cores": ""}


def run_bench(g, entries, opts, repeat=1, workers=1, **kw):
    """cli.py:128-140: every entry, input order kept; ``workers`` threads share
    the device graph (each evaluation takes its own pooled query handle)."""
    if workers <= 1:
        return [run_entry(g, e, opts, repeat, **kw) for e in entries]
    with ThreadPoolExecutor(max_workers=workers) as pool:
        return list(pool.map(lambda e: run_entry(g, e, opts, repeat, **kw), entries))


def run_batch(g, n, sources, opts, *, repeat=1, ids=None, work=True, peak_gbs=None, ngpu=1):
    """All ``sources`` through eval_ssr_batch (32 per launch); one row per
    source.  Timing follows run_entry (first of >= 2 repeats dropped, median)."""
    sources = [int(s) for s in sources]
    ids = ids or [f"s{s}" for s in sources]
    times, out, stats = [], None, []
    for r in range(max(1, repeat)):
        st = [] if r == 0 else None
        t0 = time.perf_counter()
        out = eval_ssr_batch(g, n, sources, opts, stats=st)
        times.append((time.perf_counter() - t0) * 1000.0)
        if st is not None:
            stats = st
    if len(times) >= 2:
        times = times[1:]
    total_ms = statistics.median(times)
    rows = []
    per_ms = total_ms / max(len(sources), 1)
    for i, s in enumerate(sources):
        launch = stats[i // _lib.BATCH]
        row = {"id": ids[i], "mode": "ssr", "algorithm": opts.algorithm, "result_count": int(out[i].sum()),
               "iterations": int(launch["iterations"][i % _lib.BATCH]), "time_ms": per_ms, "status": "ok"}
        if work:
            w = work_counts(g, n, s, opts)
            row.update(_ext_columns(w, per_ms, peak_gbs or read_peak_gbs(), ngpu))
        rows.append(row)
    return rows


def _fmt(v):
    if isinstance(v, float):
        return f"{v:.3f}" if abs(v) >= 1e-3 or v == 0 else f"{v:.6g}"
    return v


def write_csv(rows, out, extended=False):
    """cli.py:143-157 (time_ms with 3 decimals); ``extended`` adds EXT_HEADER's columns."""
    header = EXT_HEADER if extended else BENCH_HEADER
    w = csv.writer(out)
    w.writerow(header)
    for row in rows:
        w.writerow([_fmt(row.get(k, "")) if k != "time_ms" else f"{row['time_ms']:.3f}" for k in header])


def automaton_compiler(automata_path=None, labels=None):
    """pattern -> automaton: the reference compiler when importable, else a
    lookup in an automata JSON (``"<pattern>|min"`` keys, or plain patterns)."""
    table = {}
    if automata_path:
        with open(automata_path) as fh:
            d = json.load(fh)
        # data/config_automata.json nests per config
        flat = {}
        for k, v in d.items():
            if isinstance(v, dict) and "nstates" not in v:
                flat.update(v)
            else:
                flat[k] = v
        for k, v in flat.items():
            pat = k[:-4] if k.endswith("|min") else k
            if not k.endswith("|raw"):
                table[pat] = Automaton.from_json(v)
    if table:
        return lambda pattern: table[pattern]
    try:
        from rpq.query_compiler import compile as ref_compile
        from rpq.query_compiler import parse_query
    except ImportError as e:
        raise SystemExit("no automata JSON given and the reference compiler (rpq) is not importable") from e
    label_ids = {nm: i for i, nm in enumerate(labels or [])}
    return lambda pattern: ref_compile(parse_query(pattern), label_ids)


def _parser():
    ap = argparse.ArgumentParser(prog="paper_2412_10287_b200.cli")
    sub = ap.add_subparsers(dest="cmd", required=True)
    b = sub.add_parser("bench", help="time a workload on a synthetic BASELINE config")
    b.add_argument("--config", default="cfg1", help="synthetic graph (datagen.CONFIGS)")
    b.add_argument("--workload", help="TSV id/mode/endpoint/pattern; default: the config's query x --sources")
    b.add_argument("--automata", help="automata JSON (default: data/config_automata.json)")
    b.add_argument("--sources", type=int, default=None, help="sources per query (config's rule)")
    b.add_argument("--batch", action="store_true", help="evaluate the sources with eval_ssr_batch")
    b.add_argument("--repeat", type=int, default=3)
    b.add_argument("--workers", type=int, default=1)
    b.add_argument("--algorithm", choices=("masked", "no_mask", "hybrid"), default="hybrid")
    b.add_argument("--timeout-ms", type=float, default=math.inf)
    b.add_argument("--direction", choices=("auto", "push", "pull"), default="auto")
    b.add_argument("--plain", action="store_true", help="only the reference's 7 columns")
    b.add_argument("--out", help="CSV path (default stdout)")
    return ap


def main(argv=None):
    args = _parser().parse_args(argv)
    from . import datagen

    sg = datagen.generate(args.config)
    g = sg.labeled_graph()
    here = os.path.dirname(os.path.abspath(__file__))
    automata = args.automata or os.path.join(here, "data", "config_automata.json")
    with open(automata) as fh:
        raw = json.load(fh)
    comp_path = automata
    if args.config in raw and not args.automata:
        # only this config's automata (label indices are per config)
        import tempfile

        tmp = tempfile.NamedTemporaryFile("w", suffix=".json", delete=False)
        json.dump(raw[args.config], tmp)
        tmp.close()
        comp_path = tmp.name
    compile_fn = automaton_compiler(comp_path)
    opts = EngineOptions(algorithm=args.algorithm, timeout=args.timeout_ms / 1e3, direction=args.direction)
    peak = read_peak_gbs()
    if args.workload:
        with open(args.workload) as fh:
            entries = parse_workload(fh)
        rows = run_bench(g, entries, opts, repeat=args.repeat, workers=args.workers, compile_fn=compile_fn,
                         work=not args.plain, peak_gbs=peak)
    else:
        srcs = datagen.pick_sources(sg, args.config, count=args.sources)
        rows = []
        for qi, pattern in enumerate(datagen.CONFIGS[args.config]["queries"]):
            n = compile_fn(pattern)
            ids = [f"q{qi}-s{s}" for s in srcs]
            if args.batch:
                rows += run_batch(g, n, srcs, opts, repeat=args.repeat, ids=ids, work=not args.plain,
                                  peak_gbs=peak)
            else:
                entries = [WorkloadEntry(i, "ssr", str(s), pattern) for i, s in zip(ids, srcs)]
                rows += run_bench(g, entries, opts, repeat=args.repeat, workers=args.workers,
                                  compile_fn=lambda _p, n=n: n, work=not args.plain, peak_gbs=peak)
    out = open(args.out, "w", newline="") if args.out else sys.stdout
    try:
        write_csv(rows, out, extended=not args.plain)
    finally:
        if args.out:
            out.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
