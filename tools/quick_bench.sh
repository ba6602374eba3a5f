# quick A/B: bench lines (device GTEPS, ms/step, densest-level HBM fraction) for a few configs
for c in ${CONFIGS:-cfg2 cfg3}; do
  timeout -s KILL 600 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline $EXTRA 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$c', round(d['value'],2), round(d['ms_per_step'],4), 'dense', r.get('densest_level_frac'), ' '.join(('S' if lv['dir']=='push' else 'L')+str(int(lv['us'])) for lv in r.get('per_level', [])))"
done
