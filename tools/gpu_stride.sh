#!/bin/bash
# stage-3 throughput against the row stride (n1 * n2c * 16 bytes): same 1024-point columns, n1 = 32 .. 1024
OUT=gpurun_out/${1:-stride}
mkdir -p $OUT
for n1 in 32 64 128 256 512 1024; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file $OUT/l_$n1.csv python tools/devbench.py --shape 1024,$n1,1024 --iters 3 > $OUT/dev_$n1.txt 2>&1
done
