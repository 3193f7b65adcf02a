# ncu --set full capture of K2 (k_slice) for the given config_cell specs
# (e.g. 2_0 4_0), each after a plain run of the same command exits 0.  The
# reports are summarised on the box (tools/ncu_summary.py) and deleted unless
# KEEP=1 (gpurun_out/ must stay under 64 MiB).
mkdir -p gpurun_out/prof
keep=${KEEP:-0}
for spec in "$@"; do
  cfg=${spec%_*}; cell=${spec#*_}
  cmd="python bench.py --config $cfg --cell $cell --steps 1 --warmup 3 --no-cpu-baseline"
  timeout 900 $cmd > gpurun_out/prof/plain_c${cfg}_${cell}.log 2>&1 || { echo "plain c$spec failed"; continue; }
  rep=gpurun_out/prof/k_slice_c${cfg}_${cell}
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:${KERN:-k_slice} -s 3 -c 1 \
    -o $rep $cmd > gpurun_out/prof/ncu_c${cfg}_${cell}.log 2>&1
  echo "c$spec ncu_rc=$?"
  python tools/ncu_summary.py report $rep.ncu-rep 40 > gpurun_out/prof/sum_c${cfg}_${cell}.txt 2>&1
  [ $keep = 1 ] || rm -f $rep.ncu-rep
done
du -sh gpurun_out
