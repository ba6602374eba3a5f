#!/bin/bash
# One GPU-box pass: parity tests, bench (engine + reference arms), per-config
# sweep, batch and partitioned paths, ncu evidence.
# Usage (under gpurun): bash tools/gpu_round.sh <tag>
tag=${1:-r01}
out=gpurun_out
mkdir -p $out
timeout -s KILL 900 python -m pytest tests -q -m gpu > $out/gpu_tests_$tag.log 2>&1; echo "tests_rc=$?"; tail -3 $out/gpu_tests_$tag.log
timeout 300 python __graft_entry__.py --smoke > $out/smoke_$tag.log 2>&1; echo "smoke_rc=$?"
timeout 600 python bench.py > $out/bench_$tag.json 2> $out/bench_$tag.err; echo "bench_rc=$?"
timeout 600 python bench.py --impl reference > $out/bench_ref_$tag.json 2> $out/bench_ref_$tag.err; echo "ref_rc=$?"
timeout 900 python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu-baseline > $out/bench_cfg3_$tag.json 2> $out/bench_cfg3_$tag.err; echo "cfg3_rc=$?"
timeout 1500 python tools/config_sweep.py cfg1 cfg2 cfg3 cfg5 cfg4 --sources 8 --reps 3 > $out/sweep_$tag.jsonl 2> $out/sweep_$tag.err; echo "sweep_rc=$?"
timeout 900 python tools/batch_probe.py cfg5 --single 64 > $out/batch_cfg5_$tag.json 2> $out/batch_cfg5_$tag.err; echo "batch_rc=$?"
for qi in 0 1 2 3; do
  timeout 900 python tools/batch_probe.py cfg4 --sources 32 --single 32 --query $qi 2>/dev/null | tail -1 >> $out/batch_cfg4_$tag.jsonl
done; echo "batch4_rc=$?"
timeout 900 python -m torch.distributed.run --nnodes 1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29561 \
    tools/partition_bench.py > $out/partition_r1_$tag.json 2> $out/partition_r1_$tag.err; echo "part_rc=$?"
timeout 900 python tools/partition_bench.py --local-shards 4 > $out/partition_l4_$tag.json 2> $out/partition_l4_$tag.err; echo "part4_rc=$?"
timeout 300 python tools/trace_probe.py cfg2 > $out/trace_cfg2_$tag.jsonl 2> $out/trace_cfg2_$tag.err; echo "trace_rc=$?"
timeout 300 python bench.py --profile --steps 3 --warmup 3 > $out/prof_plain_$tag.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_$tag.csv \
    python bench.py --profile --steps 3 --warmup 3 > $out/ncu_launches_$tag.log 2>&1; echo "ncu_launch_rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ssr_kernel -s 2 -c 1 \
    -o $out/prof_cfg2_$tag python bench.py --profile --steps 3 --warmup 3 > $out/ncu_full_$tag.log 2>&1; echo "ncu_full_rc=$?"
timeout 600 python bench.py --config cfg4 --profile --steps 3 --warmup 3 > $out/prof4_plain_$tag.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:ssr_kernel -s 2 -c 1 \
    -o $out/prof_cfg4_$tag python bench.py --config cfg4 --profile --steps 3 --warmup 3 > $out/ncu4_full_$tag.log 2>&1; echo "ncu4_full_rc=$?"
timeout 600 python tools/trace_probe.py cfg4 --query 2 --max-degree --levels 30 > $out/trace_cfg4_$tag.jsonl 2> $out/trace_cfg4_$tag.err; echo "trace4_rc=$?"
