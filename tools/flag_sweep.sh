# push-path variants (RPQ_TUNE_FLAGS) across configs: GTEPS, ms per step
for c in ${CONFIGS:-cfg2 cfg3 cfg5 cfg4}; do for f in ${FLAGS:-0 1 2 3}; do
  python bench.py --steps 10 --warmup 3 --config $c --flags $f --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$c','$f',round(d['value'],2),round(d['ms_per_step'],4))"
done; done
