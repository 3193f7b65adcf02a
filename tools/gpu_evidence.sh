# Round evidence: GPU tests, the default bench line (with CPU baseline), the
# reference arm, an ncu launch list and one ncu --set full capture of K2
# (summarised on the box; gpurun_out/ must stay under 64 MiB).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/ev_pytest.log 2>&1; echo pytest_rc=$?; tail -1 gpurun_out/ev_pytest.log
timeout 900 python bench.py > gpurun_out/ev_bench.json 2> gpurun_out/ev_bench.err; echo bench_rc=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ev_ref.json 2> gpurun_out/ev_ref.err; echo ref_rc=$?
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev_launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ev_ncu_l.log 2>&1; echo ncu_l_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_slice -s 4 -c 1 -o gpurun_out/ev_k_slice \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ev_ncu_f.log 2>&1; echo ncu_f_rc=$?
python tools/ncu_summary.py report gpurun_out/ev_k_slice.ncu-rep 30 > gpurun_out/ev_k_slice_summary.txt 2>&1
python tools/ncu_summary.py launches gpurun_out/ev_launches.csv > gpurun_out/ev_launches_summary.txt 2>&1
cp profiles/traffic.json gpurun_out/traffic.json 2>/dev/null
python tools/ncu_summary.py traffic gpurun_out/ev_k_slice.ncu-rep "config2 Count-16 b=2 Levenshtein k=1" gpurun_out/traffic.json
rm -f gpurun_out/ev_k_slice.ncu-rep  # summarised above; the raw report is too large to bring back
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev_smoke.log 2>&1; echo smoke_rc=$?
du -sh gpurun_out
