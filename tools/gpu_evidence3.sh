# Round-2 evidence snapshot (K2 + K3 split): GPU tests, the default bench line
# (config 5 with e2e and the CPU baseline), the reference arm, smoke(), the
# ncu launch list of the default bench command, and ncu --set full summaries
# of the K2 sig' launch and of K3.
# usage: bash tools/gpu_evidence3.sh <tag>
tag=${1:-r02d}
o=gpurun_out/$tag; mkdir -p $o
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $o/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q > $o/pytest.log 2>&1; echo pytest_rc=$?; tail -1 $o/pytest.log
timeout 1200 python bench.py > $o/bench.json 2> $o/bench.err; echo bench_rc=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $o/ref.json 2> $o/ref.err; echo ref_rc=$?
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; echo smoke_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $o/launches.csv python bench.py --no-cpu-baseline --no-e2e --steps 1 --warmup 1 > $o/ncu_l.log 2>&1; echo ncu_l_rc=$?
python tools/ncu_summary.py launches $o/launches.csv > $o/launches_summary.txt 2>&1
bash tools/ncu_k23.sh $tag 5 0
du -sh gpurun_out
