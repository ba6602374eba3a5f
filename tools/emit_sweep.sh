set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in cfg2 cfg3 cfg5 cfg4; do for m in 0 1 2; do
  python bench.py --steps 10 --warmup 3 --config $c --emit-mode $m --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$c','$m',d['value'],d['ms_per_step'],d['roofline']['frac'])"
done; done
