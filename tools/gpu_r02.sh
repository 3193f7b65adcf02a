# Round-2 evidence run: GPU tests, ALU microbenchmark, the default bench line
# (config 5, with the CPU baseline), the reference arm, an ncu launch list
# and one ncu --set full capture of K2 (summarised on the box).
# usage: bash tools/gpu_r02.sh <tag> [skip_tests]
tag=${1:-r02a}
mkdir -p gpurun_out/$tag
o=gpurun_out/$tag
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $o/smi.txt 2>&1
if [ "${2:-}" != "skip_tests" ]; then
  timeout 900 python -m pytest tests -m gpu -q -x > $o/pytest.log 2>&1; echo pytest_rc=$?; tail -2 $o/pytest.log
fi
timeout 300 python tools/microbench/alupipe.py $tag > $o/alupipe.log 2>&1; echo alupipe_rc=$?
cp profiles/alu_peak.json $o/ 2>/dev/null; cp profiles/${tag}_alupipe.txt $o/ 2>/dev/null
timeout 1200 python bench.py > $o/bench.json 2> $o/bench.err; echo bench_rc=$?; tail -c 3000 $o/bench.json
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 1 --warmup 1 > $o/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/launches.csv \
  python bench.py --no-cpu-baseline --no-e2e --steps 1 --warmup 1 > $o/ncu_l.log 2>&1; echo ncu_l_rc=$?
python tools/ncu_summary.py launches $o/launches.csv > $o/launches_summary.txt 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_slice -s 1 -c 1 -o $o/k_slice \
  python bench.py --no-cpu-baseline --no-e2e --steps 1 --warmup 1 > $o/ncu_f.log 2>&1; echo ncu_f_rc=$?
python tools/ncu_summary.py report $o/k_slice.ncu-rep 40 > $o/k_slice_summary.txt 2>&1
python tools/ncu_summary.py sass $o/k_slice.ncu-rep > $o/k_slice_sass.txt 2>&1
ncu -i $o/k_slice.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > $o/k_slice_sass.csv.gz
rm -f $o/k_slice.ncu-rep
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $o/ref.json 2> $o/ref.err; echo ref_rc=$?
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; echo smoke_rc=$?
du -sh gpurun_out
