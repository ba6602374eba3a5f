#!/bin/bash
# A/B of engine variants on cfg3 (bench --profile: device leg only) + one ncu --set full of the heavy source.
#   bash tools/gpu_ab.sh TAG "label1|ENV=.. bench-args" "label2|..." ...
tag=$1; shift
out=gpurun_out
mkdir -p $out
for spec in "$@"; do
  label=${spec%%|*}; rest=${spec#*|}
  env $rest > /dev/null 2>&1  # validate
  eval "$rest timeout 600 python bench.py --profile --steps 5 --warmup 2" > $out/ab_${tag}_$label.json 2> $out/ab_${tag}_$label.err
  python - $out/ab_${tag}_$label.json $label <<'PY'
import json,sys
try:
    d=json.load(open(sys.argv[1]))
except Exception as e:
    print(sys.argv[2], "failed", e); sys.exit(0)
r=d["roofline"]; pl=r["per_level_heaviest_source"]
print(sys.argv[2], "value", round(d["value"],2), "ms/step", round(d["ms_per_step"],3), "levels_us", [l["us"] for l in pl])
PY
done
