# One ncu --set full capture of K2 (k_slice) on a config cell, summarised on
# the box, plus the ncu launch list of the same bench command.
# usage: bash tools/ncu_cell.sh <tag> <cfg> <cell> [extra env]
tag=$1; cfg=$2; cell=$3; shift 3
o=gpurun_out/$tag; mkdir -p $o
env "$@" timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:${KREGEX:-k_slice}" -s 1 -c 1 -o $o/k_slice \
    python bench.py --config $cfg --cell $cell --no-cpu-baseline --no-e2e --steps 1 --warmup 1 > $o/ncu_f.log 2>&1
echo ncu_rc=$?
python tools/ncu_summary.py report $o/k_slice.ncu-rep 40 > $o/k_slice_summary.txt 2>&1
python tools/ncu_summary.py sass $o/k_slice.ncu-rep > $o/k_slice_sass.txt 2>&1
ncu -i $o/k_slice.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > $o/k_slice_sass.csv.gz
key=$(python -c "import bench; w=bench.Workload.__new__(bench.Workload); w.cfg, w.cell = $cfg, $cell; print('config$cfg', w.cell_name())")
python tools/ncu_summary.py traffic $o/k_slice.ncu-rep "$key" $o/traffic.json > /dev/null 2>&1
rm -f $o/k_slice.ncu-rep
env "$@" timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $o/launches.csv \
  python bench.py --config $cfg --cell $cell --no-cpu-baseline --no-e2e --steps 1 --warmup 1 > $o/ncu_l.log 2>&1; echo ncu_l_rc=$?
python tools/ncu_summary.py launches $o/launches.csv > $o/launches_summary.txt 2>&1
