OUT=gpurun_out/exp4; mkdir -p $OUT
for pr in 0 1 2 3; do
TFFFT_PROBE_COL=$pr ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/probe$pr.csv python tools/devbench.py --n 1024 --iters 2 > /dev/null 2>&1
done
