OUT=gpurun_out/exp2; mkdir -p $OUT
CMD="python tools/devbench.py --n 1024 --iters 5"
$CMD > $OUT/base.txt 2>&1
TFFFT_PROBE_ALIAS=1 $CMD > $OUT/alias.txt 2>&1
TFFFT_PROBE_ALIAS=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/alias_launches.csv $CMD > /dev/null 2>&1
