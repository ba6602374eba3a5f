#!/bin/bash
# Round-2 first GPU pass: tests, cfg3 headline bench (both arms), ncu of cfg3.
tag=${1:-r02a}
out=gpurun_out
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $out/smi_$tag.txt 2>&1
timeout -s KILL 1200 python -m pytest tests -q -m gpu -x > $out/gpu_tests_$tag.log 2>&1; echo "tests_rc=$?"; tail -3 $out/gpu_tests_$tag.log
timeout 300 python __graft_entry__.py --smoke > $out/smoke_$tag.log 2>&1; echo "smoke_rc=$?"
timeout 900 python bench.py > $out/bench_$tag.json 2> $out/bench_$tag.err; echo "bench_rc=$?"
timeout 900 python bench.py --impl reference > $out/bench_ref_$tag.json 2> $out/bench_ref_$tag.err; echo "ref_rc=$?"
timeout 600 python bench.py --profile --steps 1 --warmup 1 > $out/prof_plain_$tag.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_$tag.csv \
    python bench.py --profile --steps 1 --warmup 1 > $out/ncu_launches_$tag.log 2>&1; echo "ncu_launch_rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ssr_kernel -s 1 -c 1 \
    -o $out/prof_cfg3_$tag python bench.py --profile --steps 1 --warmup 0 --source 6658600 > $out/ncu_full_$tag.log 2>&1; echo "ncu_full_rc=$?"
