# Every feasible cell of every config through bench.py (1 GPU, short runs, no CPU baseline).
mkdir -p gpurun_out/sweep
for cfg in 1 2 3 4 5; do
  n=$(python -c "from paper_1711_08475_b200.corpus import CELLS; print(len(CELLS[$cfg]))")
  for ((cell=0; cell<n; cell++)); do
    steps=5; [ $cfg -ge 3 ] && steps=3
    timeout 900 python bench.py --config $cfg --cell $cell --steps $steps --warmup 3 --no-cpu-baseline \
      > gpurun_out/sweep/c${cfg}_${cell}.log 2>&1
    echo "cfg=$cfg cell=$cell rc=$? $(tail -1 gpurun_out/sweep/c${cfg}_${cell}.log | python -c 'import sys,json
try:
  d=json.loads(sys.stdin.read()); r=d["roofline"]; v=d.get("verify") or {}
  print(d["config"]["cell"], "step_ms=%.3f" % d["ms_per_step"], "k2_ms=%.3f" % r["filter_ms_per_launch"], "k3_ms=%.3f" % v.get("ms_per_step", 0), "Tcmp/s=%.2f" % r["achieved"], "frac=%.2f" % r["frac"], "popc_frac=%.2f" % r["popc_equiv_frac"], "e2e=%.3g" % d["e2e"]["value"], "matches=%d" % d["matches_per_step"], "cand=%d" % d["verifier_candidates_per_step"])
except Exception as e: print("parse error", e)')"
  done
done
