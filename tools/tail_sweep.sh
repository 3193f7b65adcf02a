# A/B of the K2 tail-splitting fractions (FPG_TAIL_A / FPG_TAIL_B) on config 2.
for ab in "0.35 0.85" "0.2 0.7"; do
  set -- $ab
  FPG_TAIL_A=$1 FPG_TAIL_B=$2 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$1 $2', d['ms_per_step'], d['roofline']['filter_ms_per_launch'])"
done
