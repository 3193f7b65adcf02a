# A/B of environment switches on a bench cell.  usage: bash tools/ab_k3.sh <cfg> <cell> VAR=val [VAR=val ...]  (one run per setting)
cfg=$1; cell=$2; shift 2
for v in "$@"; do
  env $v FPG_VERIFY_CTAS=592 python bench.py --config $cfg --cell $cell --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print('$v', 'step %.2f' % d['ms_per_step'], 'k2 %.2f' % d['roofline']['filter_ms_per_launch'], 'k3 %.2f' % d['verify']['ms_per_step'], 'frac %.3f' % d['roofline']['frac'])"
done
