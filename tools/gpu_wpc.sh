#!/bin/bash
# A/B of the warp-per-column kernel on one box
OUT=gpurun_out/${1:-wpc}
mkdir -p $OUT
timeout 300 python tools/wpc_check.py > $OUT/check.txt 2>&1; echo "check exit $?" >> $OUT/check.txt
if grep -q "ALL OK" $OUT/check.txt; then
for rep in 1 2; do
for m in 0 1; do
  echo "== TFFFT_WPC=$m f64" >> $OUT/ab.txt
  TFFFT_WPC=$m timeout 300 python tools/devbench.py --n 1024 --iters 10 >> $OUT/ab.txt 2>&1
done
done
for m in 0 1; do
  echo "== TFFFT_WPC=$m f32" >> $OUT/ab.txt
  TFFFT_WPC=$m timeout 300 python tools/devbench.py --n 1024 --dtype float32 --iters 10 >> $OUT/ab.txt 2>&1
done
for m in 0 1; do
TFFFT_WPC=$m timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file $OUT/launches_wpc$m.csv python tools/devbench.py --n 1024 --iters 2 > /dev/null 2>&1
done
fi
