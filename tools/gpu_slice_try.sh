mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pt_slice.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pt_slice.log
for S in 16; do FPG_SIGP_BITS=$S timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bs_$S.log 2>&1; echo S=$S rc=$?; tail -1 gpurun_out/bs_$S.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['filter_ms_per_launch'], d['matches_per_step'], d['verifier_candidates_per_step'], d['e2e']['value'], d['gpu_launches'])" ; done
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_slice -s 4 -c 1 -o gpurun_out/r01_k_slice_c python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_f.log 2>&1; echo ncuf_rc=$?
