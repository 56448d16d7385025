#!/bin/bash
# 2048-point column kernel at BASELINE config 4's per-rank sizes (2048^3 / 8): launch lists + one full capture
OUT=gpurun_out/${1:-l11f}
mkdir -p $OUT
for sh in "256,2048,2048" "2048,256,2048"; do
  echo "== $sh" >> $OUT/dev.txt
  timeout 300 python tools/devbench.py --shape $sh --iters 5 >> $OUT/dev.txt 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file $OUT/launches_$(echo $sh | tr ',' 'x').csv python tools/devbench.py --shape $sh --iters 1 > /dev/null 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:col_wpc2 -s 2 -c 1 -o $OUT/wpc2 \
    python tools/devbench.py --shape 256,2048,2048 --iters 1 > $OUT/ncu_full.log 2>&1
