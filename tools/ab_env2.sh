# A/B of "VAR=val,VAR2=val2" settings on a bench cell (one run per setting).
# usage: bash tools/ab_env2.sh <cfg> <cell> <steps> "A=1,B=2" "A=3" ...
cfg=$1; cell=$2; steps=$3; shift 3
for v in "$@"; do
  env $(echo $v | tr ',' ' ') python bench.py --config $cfg --cell $cell --steps $steps --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print('$v', 'step %.4f' % d['ms_per_step'], 'k2 %.4f' % d['roofline']['filter_ms_per_launch'], 'k3 %.4f' % (d['verify'] or {}).get('ms_per_step',0), 'frac %.3f' % d['roofline']['frac'])"
done
