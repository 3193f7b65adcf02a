o=gpurun_out/r02h; mkdir -p $o
FPG_DROP_CANDIDATES=1 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_slice -s 1 -c 1 -o $o/k_slice \
    python bench.py --config 5 --cell 0 --no-cpu-baseline --no-e2e --steps 1 --warmup 1 > $o/ncu_f.log 2>&1
echo ncu_rc=$?
python tools/ncu_summary.py report $o/k_slice.ncu-rep 40 > $o/k_slice_summary.txt 2>&1
ncu -i $o/k_slice.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > $o/k_slice_sass.csv.gz
rm -f $o/k_slice.ncu-rep
