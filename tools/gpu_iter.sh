# Iteration run: GPU tests, bench lines for the given config_cell specs
# (no CPU baseline, no e2e), and optionally one ncu --set full capture of K2
# on the first spec (NCU=1), summarised on the box.
# usage: bash tools/gpu_iter.sh <tag> <cfg_cell> [<cfg_cell> ...]
tag=$1; shift
o=gpurun_out/$tag; mkdir -p $o
if [ "${TESTS:-1}" = 1 ]; then
  timeout 900 python -m pytest tests -m gpu -q -x > $o/pytest.log 2>&1; echo pytest_rc=$?; tail -1 $o/pytest.log
fi
for spec in "$@"; do
  cfg=${spec%_*}; cell=${spec#*_}
  timeout 900 python bench.py --config $cfg --cell $cell --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --no-e2e \
    > $o/b_c${spec}.json 2> $o/b_c${spec}.err; echo "c$spec rc=$?"
  python - "$o/b_c${spec}.json" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r = d["roofline"]
    print(d["config"]["cell"], "step_ms=%.3f" % d["ms_per_step"], "k2_ms=%.3f" % r["filter_ms_per_launch"],
          "value=%.4g" % d["value"], "frac=%.3f" % r["frac"], "eval=%.4g" % d["evaluated_pairs_per_step"],
          "cand=%d" % d["verifier_candidates_per_step"], "matches=%s" % d["matches_per_step"])
except Exception as e:
    print("parse error", e)
PY
done
if [ "${NCU:-0}" = 1 ]; then
  spec=$1; cfg=${spec%_*}; cell=${spec#*_}
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_slice -s 1 -c 1 -o $o/k_slice \
    python bench.py --config $cfg --cell $cell --no-cpu-baseline --no-e2e --steps 1 --warmup 1 > $o/ncu_f.log 2>&1
  echo ncu_rc=$?
  python tools/ncu_summary.py report $o/k_slice.ncu-rep 40 > $o/k_slice_summary.txt 2>&1
  python tools/ncu_summary.py sass $o/k_slice.ncu-rep > $o/k_slice_sass.txt 2>&1
  ncu -i $o/k_slice.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > $o/k_slice_sass.csv.gz
  rm -f $o/k_slice.ncu-rep
fi
du -sh gpurun_out
