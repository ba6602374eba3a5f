#!/bin/bash
# A/B of engine variants (bench --profile: device leg only).
#   bash tools/gpu_ab.sh TAG "label|ENV=.. ENV2=..|bench args" ...
tag=$1; shift
out=gpurun_out
mkdir -p $out
for spec in "$@"; do
  label=${spec%%|*}; rest=${spec#*|}; envs=${rest%%|*}; args=${rest#*|}
  env $envs timeout 600 python bench.py --profile --steps 5 --warmup 2 $args > $out/ab_${tag}_$label.json 2> $out/ab_${tag}_$label.err
  python - $out/ab_${tag}_$label.json $label <<'PY'
import json,sys
try:
    d=json.load(open(sys.argv[1]))
except Exception as e:
    print(sys.argv[2], "failed", e); sys.exit(0)
r=d["roofline"]; pl=r["per_level_heaviest_source"]
print(sys.argv[2], d["config"]["workload"][:5], "value", round(d["value"],2), "ms/step", round(d["ms_per_step"],3), "levels_us", [l["us"] for l in pl])
PY
done
