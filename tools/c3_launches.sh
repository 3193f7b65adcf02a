for cell in 0 1; do
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_$cell.csv python bench.py --config 3 --cell $cell --no-cpu-baseline --no-e2e --steps 2 --warmup 1 > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/c3_$cell.csv | head -14
done
