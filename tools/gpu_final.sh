#!/bin/bash
# Round-end evidence: GPU suite, smoke, the default bench (engine + reference
# arms), the launch list and one ncu --set full capture of the heaviest cfg3
# query, the cfg5 batch bench and its capture, the partitioned mode.
tag=${1:-final}
out=gpurun_out
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $out/smi_$tag.txt 2>&1
timeout -s KILL 1500 python -m pytest tests -q -m gpu -x > $out/gpu_tests_$tag.log 2>&1; echo "tests_rc=$?"; tail -2 $out/gpu_tests_$tag.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke_$tag.log 2>&1; echo "smoke_rc=$?"; tail -1 $out/smoke_$tag.log
timeout 900 python bench.py > $out/bench_$tag.json 2> $out/bench_$tag.err; echo "bench_rc=$?"
timeout 900 python bench.py --impl reference > $out/bench_ref_$tag.json 2> $out/bench_ref_$tag.err; echo "ref_rc=$?"
timeout 900 python bench.py --mode batch --config cfg5 --steps 3 --warmup 1 > $out/bench_batch_$tag.json 2> $out/bench_batch_$tag.err; echo "batch_rc=$?"
timeout 900 python bench.py --mode partitioned --steps 3 --warmup 1 > $out/bench_part_$tag.json 2> $out/bench_part_$tag.err; echo "part_rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_$tag.csv \
    python bench.py --profile --steps 1 --warmup 1 > $out/ncu_launches_$tag.log 2>&1; echo "ncu_launch_rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ssr_kernel -s 1 -c 1 \
    -o $out/prof_cfg3_$tag python bench.py --profile --steps 1 --warmup 0 --source 10754584 > $out/ncu_full_$tag.log 2>&1; echo "ncu_full_rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:batch_kernel -s 3 -c 1 \
    -o $out/prof_batch_$tag python bench.py --mode batch --config cfg5 --profile --steps 1 --warmup 0 --sources 192 > $out/ncu_batch_$tag.log 2>&1; echo "ncu_batch_rc=$?"
python - $out $tag <<'PY'
import json, sys
out, tag = sys.argv[1], sys.argv[2]
for f in ("bench", "bench_ref", "bench_batch", "bench_part"):
    try:
        d = json.load(open(f"{out}/{f}_{tag}.json"))
        e = d.get("e2e", {})
        print(f, round(d["value"], 2), "e2e", round(e.get("value", 0), 2) if e else None,
              "frac", d.get("roofline", {}).get("frac"), d.get("roofline", {}).get("densest_level_frac"))
    except Exception as ex:
        print(f, "unreadable", ex)
PY
