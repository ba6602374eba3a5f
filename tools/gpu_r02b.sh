#!/bin/bash
# Round-2 probe: new GPU tests (CLI), cfg3 per-level trace, e2e breakdowns, sanitizers.
tag=${1:-r02b}
out=gpurun_out
mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_cli.py -q -x > $out/gpu_cli_$tag.log 2>&1; echo "cli_tests_rc=$?"; tail -3 $out/gpu_cli_$tag.log
timeout 600 python tools/trace_probe.py cfg3 --levels 12 > $out/trace_cfg3_$tag.jsonl 2>&1; echo "trace_rc=$?"
timeout 600 python tools/e2e_probe.py cfg3 10754584 > $out/e2e_cfg3_heavy_$tag.txt 2>&1; echo "e2e_heavy_rc=$?"
timeout 600 python tools/e2e_probe.py cfg3 13177147 > $out/e2e_cfg3_empty_$tag.txt 2>&1; echo "e2e_empty_rc=$?"
bash tools/gpu_sanitize.sh $tag
