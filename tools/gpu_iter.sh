#!/bin/bash
# One build->measure iteration on the GPU box: GPU tests, cfg3 bench (engine
# arm, no CPU baseline), per-level trace of the first cfg3 source, e2e split.
#   bash tools/gpu_iter.sh TAG [tests|notests]
tag=${1:-iter}
out=gpurun_out
mkdir -p $out
if [ "${2:-tests}" = tests ]; then
  timeout -s KILL 1500 python -m pytest tests -q -m gpu -x > $out/gpu_tests_$tag.log 2>&1; echo "tests_rc=$?"; tail -3 $out/gpu_tests_$tag.log
fi
timeout 900 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > $out/bench_$tag.json 2> $out/bench_$tag.err; echo "bench_rc=$?"
python - $out/bench_$tag.json <<'PY'
import json,sys
try:
    d=json.load(open(sys.argv[1]))
except Exception as e:
    print("bench parse failed", e); sys.exit(0)
r=d["roofline"]
print("value", round(d["value"],2), "e2e", round(d.get("e2e",{}).get("value",0),2), "frac", round(r["frac"],4), "dense", r["densest_level_frac"])
print("lat", {k: round(v,4) for k,v in d["per_query"]["latency_ms_median"].items()})
for l in r["per_level_heaviest_source"]: print(" ", l)
PY
timeout 600 python tools/trace_probe.py cfg3 --levels 12 --source 10754584 > $out/trace_cfg3_$tag.jsonl 2>&1; echo "trace_rc=$?"
timeout 600 python tools/e2e_split.py cfg3 10754584 13177147 > $out/e2e_split_$tag.txt 2>&1; echo "e2e_rc=$?"; cat $out/e2e_split_$tag.txt
