set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/r01_pytest_gpu.log 2>&1; echo pytest_rc=$?
python bench.py --steps 50 --warmup 3 > gpurun_out/r01_bench_v1.log 2>&1; echo bench_rc=$?
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches_v1.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_l.log 2>&1; echo ncu_rc=$?
ncu --set full --clock-control none --import-source on -k regex:k_scan -s 4 -c 1 -o gpurun_out/r01_k_scan_v1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_f.log 2>&1; echo ncuf_rc=$?
tail -3 gpurun_out/r01_pytest_gpu.log; tail -1 gpurun_out/r01_bench_v1.log
