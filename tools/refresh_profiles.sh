#!/bin/bash
# Copy one gpu_round.sh pass (tag) from gpurun_out/ into profiles/ and derive
# the ncu summaries.  Usage: bash tools/refresh_profiles.sh r01d
G=gpurun_out; T=${1:?tag}
cp $G/bench_$T.json profiles/r01_bench_cfg2.json
cp $G/bench_ref_$T.json profiles/r01_bench_reference_arm.json
cp $G/bench_cfg3_$T.json profiles/r01_bench_cfg3.json
cp $G/sweep_$T.jsonl profiles/r01_config_sweep.jsonl
cp $G/batch_cfg5_$T.json profiles/r01_cfg5_batch_probe.json
cp $G/batch_cfg4_$T.jsonl profiles/r01_cfg4_batch_probe.jsonl
grep '^{' $G/partition_r1_$T.json > profiles/r01_cfg3_partition_ranks1.json
grep '^{' $G/partition_l4_$T.json > profiles/r01_cfg3_partition_local4.json
cp $G/launches_$T.csv profiles/r01_cfg2_launches.csv
cp $G/trace_cfg2_$T.jsonl profiles/r01_cfg2_trace.jsonl
cp $G/gpu_tests_$T.log profiles/r01_gpu_tests.log
ncu -i $G/prof_cfg2_$T.ncu-rep --page details --csv > profiles/r01_cfg2_ssr_kernel_details.csv 2>/dev/null
# (cfg2 runs the 768-thread instance, cfg4 the 1,024-thread one)
python tools/ncu_lines.py $G/prof_cfg2_$T.ncu-rep paper_2412_10287_b200/librpq_b200.so ssr_kernelILi768 > profiles/r01_cfg2_stall_lines.txt 2>&1
if [ -f $G/prof_cfg4_$T.ncu-rep ]; then
  ncu -i $G/prof_cfg4_$T.ncu-rep --page details --csv > profiles/r01_cfg4_ssr_kernel_details.csv 2>/dev/null
  python tools/ncu_lines.py $G/prof_cfg4_$T.ncu-rep paper_2412_10287_b200/librpq_b200.so ssr_kernelILi1024 > profiles/r01_cfg4_stall_lines.txt 2>&1
  cp $G/trace_cfg4_$T.jsonl profiles/r01_cfg4_trace.jsonl
fi
ncu -i $G/prof_cfg2_$T.ncu-rep --page raw --csv 2>/dev/null | T=$T python -c "
import csv, json, os, sys
r = list(csv.reader(sys.stdin)); h, u, v = r[0], r[1], r[2]
def val(k):
    i = h.index(k); x = float(v[i].replace(',', ''))
    return x * {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9}.get(u[i], 1)
d = {'cfg2': {'dram_bytes_per_launch': val('dram__bytes_read.sum') + val('dram__bytes_write.sum'),
              'duration_us': val('gpu__time_duration.sum') if u[h.index('gpu__time_duration.sum')] != 'us' else float(v[h.index('gpu__time_duration.sum')]),
              'l2_hit_pct': float(v[h.index('lts__t_sector_hit_rate.pct')]),
              'source': 'ncu --set full, profiles/r01_cfg2_ssr_kernel_details.csv (tools/gpu_round.sh ' + os.environ['T'] + ')'}}
json.dump(d, open('profiles/ncu_dram_bytes.json', 'w'), indent=1); print(d)"
