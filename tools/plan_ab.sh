# A/B of the K2 tile shape for small batches on config 2: PLANS="gpw,q ..." (FPG_TILE_GPW / FPG_TILE_Q).
mkdir -p gpurun_out/ab
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/ab/pt.log 2>&1; echo pytest_rc=$?; tail -1 gpurun_out/ab/pt.log
for v in ${PLANS:-2,32 4,16 4,32 1,64}; do set -- ${v/,/ }
  FPG_TILE_GPW=$1 FPG_TILE_Q=$2 timeout 300 python bench.py --config 2 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ab/c2_$1_$2.log 2>&1
  echo "gpw=$1 q=$2 $(tail -1 gpurun_out/ab/c2_$1_$2.log | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print("step_ms=%.4f k2_ms=%.4f e2e=%.3g" % (d["ms_per_step"], d["roofline"]["filter_ms_per_launch"], d["e2e"]["value"]))')"
done
