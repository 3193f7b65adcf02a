# Short bench runs of the given config_cell specs (no tests).  usage: bash tools/gpu_bench_only.sh 5_0 2_0 ...
mkdir -p gpurun_out/sweep
for spec in "$@"; do
  cfg=${spec%_*}; cell=${spec#*_}
  timeout 900 python bench.py --config $cfg --cell $cell --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/sweep/c${cfg}_${cell}.log 2>&1
  echo "cfg=$cfg cell=$cell rc=$? $(tail -1 gpurun_out/sweep/c${cfg}_${cell}.log | python -c 'import sys,json
try:
  d=json.loads(sys.stdin.read()); r=d["roofline"]; v=d.get("verify") or {}
  print(d["config"]["cell"], "step_ms=%.3f" % d["ms_per_step"], "k2_ms=%.3f" % r["filter_ms_per_launch"], "k3_ms=%.3f" % v.get("ms_per_step", 0), "Tcmp/s=%.2f" % r["achieved"], "frac=%.2f" % r["frac"], "eval/exec=%.3f" % (d["evaluated_pairs_per_step"] / max(1, d["executed_pairs_per_step"])), "e2e=%.3g" % d["e2e"]["value"], "matches=%d" % d["matches_per_step"], "cand=%d" % d["verifier_candidates_per_step"])
except Exception as e: print("parse error", e)')"
done
