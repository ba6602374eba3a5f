#!/bin/bash
# Partitioned and batch bench modes + the partition tests.
tag=${1:-modes}
out=gpurun_out
mkdir -p $out
timeout -s KILL 900 python -m pytest tests/test_gpu_partition.py tests/test_gpu_output.py -q -x > $out/gpu_part_tests_$tag.log 2>&1; echo "tests_rc=$?"; tail -3 $out/gpu_part_tests_$tag.log
NCCL_DEBUG=INFO timeout 900 python bench.py --mode partitioned --steps 5 --warmup 2 > $out/bench_part_$tag.json 2> $out/bench_part_$tag.err; echo "part_rc=$?"; tail -c 1500 $out/bench_part_$tag.json; grep -i "nccl" $out/bench_part_$tag.err | head -5
timeout 900 python bench.py --mode batch --config cfg5 --steps 3 --warmup 1 > $out/bench_batch_$tag.json 2> $out/bench_batch_$tag.err; echo "batch_rc=$?"; head -c 600 $out/bench_batch_$tag.json; echo
timeout 900 python bench.py --mode batch --config cfg5 --automaton raw --steps 3 --warmup 1 > $out/bench_batchraw_$tag.json 2> $out/bench_batchraw_$tag.err; echo "batchraw_rc=$?"; head -c 600 $out/bench_batchraw_$tag.json; echo
tail -5 $out/bench_batch_$tag.err
