for g in 32 64 128; do
  for spec in 5_0 2_0; do
    cfg=${spec%_*}; cell=${spec#*_}
    FPG_TILE_GROUPS=$g timeout 600 python bench.py --config $cfg --cell $cell --steps 5 --warmup 2 --no-cpu-baseline --no-e2e > /tmp/o.json 2>/dev/null
    python -c "
import json; d=json.loads(open('/tmp/o.json').read().strip().splitlines()[-1]); r=d['roofline']
print('groups=$g c$spec', 'step_ms=%.3f'%d['ms_per_step'], 'k2=%.3f'%r['filter_ms_per_launch'], 'frac=%.3f'%r['frac'])"
  done
done
