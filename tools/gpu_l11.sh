#!/bin/bash
# column kernels at 2048 / 4096 points (BASELINE config 4's per-rank shapes)
OUT=gpurun_out/${1:-l11}
mkdir -p $OUT
for sh in "2048,2048,64" "2048,64,2048" "64,2048,2048" "4096,1024,32"; do
  echo "== $sh" >> $OUT/dev.txt
  timeout 300 python tools/devbench.py --shape $sh --iters 5 >> $OUT/dev.txt 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file $OUT/launches_$(echo $sh | tr ',' 'x').csv python tools/devbench.py --shape $sh --iters 1 > /dev/null 2>&1
done
