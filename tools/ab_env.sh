# A/B of run-time switches: for each "VAR=value" setting (or "-" for none)
# and each config_cell, one bench line (no CPU baseline, no e2e).
# usage: bash tools/ab_env.sh <tag> "<settings...>" <cfg_cell> [<cfg_cell> ...]
tag=$1; settings=$2; shift 2
o=gpurun_out/$tag; mkdir -p $o
for st in $settings; do
  for spec in "$@"; do
    cfg=${spec%_*}; cell=${spec#*_}
    if [ "$st" = "-" ]; then envs=""; else envs="$st"; fi
    env $envs timeout 900 python bench.py --config $cfg --cell $cell --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --no-e2e \
      > $o/b_${st//=/_}_c$spec.json 2> $o/b_${st//=/_}_c$spec.err
    python - "$o/b_${st//=/_}_c$spec.json" "$st" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r = d["roofline"]
    print(sys.argv[2], d["config"]["workload"], d["config"]["cell"], "step_ms=%.3f" % d["ms_per_step"], "k2_ms=%.3f" % r["filter_ms_per_launch"],
          "frac=%.3f" % r["frac"], "cand=%d" % d["verifier_candidates_per_step"], "matches=%s" % d["matches_per_step"])
except Exception as e:
    print(sys.argv[2], "parse error", e)
PY
  done
done
