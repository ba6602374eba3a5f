#!/bin/bash
# Final verification of the shipped tree: the GPU suite on both builds, smoke,
# the default bench line (engine arm), and every BASELINE config on one GPU.
tag=${1:-verify}
out=gpurun_out
mkdir -p $out
timeout -s KILL 1500 python -m pytest tests -q -m gpu -x > $out/gpu_tests_$tag.log 2>&1; echo "tests_rc=$?"; tail -2 $out/gpu_tests_$tag.log
RPQ_ENGINE=checked timeout -s KILL 1800 python -m pytest tests -q -m gpu -x -p no:cacheprovider > $out/gpu_tests_checked_$tag.log 2>&1; echo "checked_rc=$?"; tail -2 $out/gpu_tests_checked_$tag.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke_$tag.log 2>&1; echo "smoke_rc=$?"; tail -1 $out/smoke_$tag.log
timeout 900 python bench.py > $out/bench_$tag.json 2> $out/bench_$tag.err; echo "bench_rc=$?"
timeout 1500 python tools/config_sweep.py cfg1 cfg2 cfg3 cfg4 cfg5 > $out/sweep_$tag.jsonl 2> $out/sweep_$tag.err; echo "sweep_rc=$?"
python - $out $tag <<'PY'
import json, sys
out, tag = sys.argv[1], sys.argv[2]
d = json.load(open(f"{out}/bench_{tag}.json"))
print("bench", round(d["value"], 2), "e2e", round(d["e2e"]["value"], 2), "frac", round(d["roofline"]["frac"], 4),
      d["roofline"]["densest_level_frac"], "traffic", d["roofline"]["traffic"])
for ln in open(f"{out}/sweep_{tag}.jsonl"):
    try:
        r = json.loads(ln)
        print(r.get("config"), r.get("query"), round(r.get("gteps", 0), 2), r.get("latency_ms_median"))
    except Exception:
        pass
PY
