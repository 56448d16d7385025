OUT=gpurun_out/exp10; mkdir -p $OUT
for d in 0 2000 4000; do
TFFFT_PROBE_COL=$((d*256)) ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/d$d.csv python tools/devbench.py --n 1024 --iters 2 > /dev/null 2>&1
done
