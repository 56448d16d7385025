#!/bin/bash
# quick A/B: devbench (live) at 1024^3 f64 x3 + ncu launch list of one pair
OUT=gpurun_out/${1:-q}
mkdir -p $OUT
shift
for rep in 1 2 3; do
  timeout 300 python tools/devbench.py --n 1024 --iters 10 "$@" >> $OUT/devbench.txt 2>&1
done
CMD="python tools/devbench.py --n 1024 --iters 1 $*"
WARM=1 $CMD > /dev/null 2>&1 && WARM=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/launches.csv $CMD > /dev/null 2>&1
echo "ncu $?" >> $OUT/devbench.txt
