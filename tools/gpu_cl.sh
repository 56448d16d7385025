#!/bin/bash
# A/B: col_tma_kernel stage 3 as clusters of C CTAs on consecutive tiles, boxes issued behind a cluster barrier
OUT=gpurun_out/cl; mkdir -p $OUT
for c in 1 2 4 8; do
  echo "== TFFFT_S3_CLUSTER=$c" >> $OUT/live.txt
  TFFFT_S3_CLUSTER=$c timeout 200 python tools/devbench.py --n 1024 --iters 20 --check >> $OUT/live.txt 2>&1
  echo "exit $?" >> $OUT/live.txt
done
for c in 1 2 4 8; do
  TFFFT_S3_CLUSTER=$c timeout 400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $OUT/launches_cl$c.csv python tools/devbench.py --n 1024 --iters 3 > $OUT/ncu$c.log 2>&1
  echo "== TFFFT_S3_CLUSTER=$c" >> $OUT/launches.txt
  python tools/launch_summary.py $OUT/launches_cl$c.csv | grep -E "col_tma|col_wpc" >> $OUT/launches.txt 2>&1
done
echo "== TFFFT_S3_CLUSTER=1 again" >> $OUT/live.txt
TFFFT_S3_CLUSTER=1 timeout 200 python tools/devbench.py --n 1024 --iters 20 >> $OUT/live.txt 2>&1
