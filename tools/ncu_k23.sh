# ncu --set full captures of the K2 sig' launch (k_slice, not the exact path)
# and of K3 (k_verify) on a config cell, summarised on the box.
# usage: bash tools/ncu_k23.sh <tag> <cfg> <cell> [extra env]
tag=$1; cfg=$2; cell=$3; shift 3
o=gpurun_out/$tag; mkdir -p $o
run="python bench.py --config $cfg --cell $cell --no-cpu-baseline --no-e2e --steps 1 --warmup 1"
for k in ${KERNELS:-k_verify k_slice}; do
  # default: the sig' launch (X = 0, NB = 0); KREGEX=k_slice takes the batch's second K2 launch whatever it is
  re=$k; [ $k = k_slice ] && re=${KREGEX:-'k_slice.*bool.0, .bool.0>'}
  env "$@" timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$re" -s 1 -c 1 -o $o/$k $run > $o/ncu_$k.log 2>&1
  echo ${k}_ncu_rc=$?
  python tools/ncu_summary.py report $o/$k.ncu-rep 40 > $o/${k}_summary.txt 2>&1
  python tools/ncu_summary.py sass $o/$k.ncu-rep > $o/${k}_sass.txt 2>&1
  ncu -i $o/$k.ncu-rep --page details --csv 2>/dev/null | gzip > $o/${k}_details.csv.gz
  ncu -i $o/$k.ncu-rep --page raw --csv 2>/dev/null | gzip > $o/${k}_raw.csv.gz
  key=$(python -c "import bench; w=bench.Workload.__new__(bench.Workload); w.cfg, w.cell = $cfg, $cell; print('config$cfg', w.cell_name())")
  [ $k = k_verify ] && key="$key k_verify"
  python tools/ncu_summary.py traffic $o/$k.ncu-rep "$key" $o/traffic.json > /dev/null 2>&1
  rm -f $o/$k.ncu-rep
done
