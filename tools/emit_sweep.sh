# emission placement (RPQ_TUNE_EMIT_MODE / _INLINE_MAX) across configs
for c in ${CONFIGS:-cfg2 cfg3 cfg5 cfg4}; do for m in ${MODES:-"0 0" "2 2048" "2 8192" "2 32768"}; do
  set -- $m
  python bench.py --steps 10 --warmup 3 --config $c --emit-mode $1 --emit-inline-max $2 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$c','$1','$2',round(d['value'],2),round(d['ms_per_step'],4))"
done; done
