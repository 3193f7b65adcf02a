# sig' field count A/B on the given config_cell specs: FPG_SIGP_BITS in {0, 8, 12, 16}.
mkdir -p gpurun_out/sigp
for spec in "$@"; do
  cfg=${spec%_*}; cell=${spec#*_}
  for sb in ${SBS:-0 8 12 16}; do
    FPG_SIGP_BITS=$sb timeout 900 python bench.py --config $cfg --cell $cell --steps 3 --warmup 3 --no-cpu-baseline \
      > gpurun_out/sigp/c${cfg}_${cell}_s$sb.log 2>&1
    echo "c$spec S=$sb $(tail -1 gpurun_out/sigp/c${cfg}_${cell}_s$sb.log | python -c 'import sys,json
try:
  d=json.loads(sys.stdin.read()); r=d["roofline"]; print("step_ms=%.3f k2_ms=%.3f cand=%d" % (d["ms_per_step"], r["filter_ms_per_launch"], d["verifier_candidates_per_step"]))
except Exception as e: print("parse error", e)')"
  done
done
