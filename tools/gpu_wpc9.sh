#!/bin/bash
# 512-point columns on the warp-per-column kernel: same-box A/B (live pair + ncu launch list); 1024^3 regression check
OUT=gpurun_out/${1:-wpc9}
mkdir -p $OUT
for rep in 1 2; do
for m in 0 2; do
  echo "== TFFFT_WPC=$m 512^3 f64 rep $rep" >> $OUT/ab.txt
  TFFFT_WPC=$m timeout 300 python tools/devbench.py --n 512 --iters 50 >> $OUT/ab.txt 2>&1
done
done
for m in 0 2; do
  echo "== TFFFT_WPC=$m 512^3 f32" >> $OUT/ab.txt
  TFFFT_WPC=$m timeout 300 python tools/devbench.py --n 512 --dtype float32 --iters 50 >> $OUT/ab.txt 2>&1
done
for m in 0 2; do
  TFFFT_WPC=$m timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
     --log-file $OUT/launches_512_wpc$m.csv python tools/devbench.py --n 512 --iters 2 > /dev/null 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
     --log-file $OUT/launches_1024.csv python tools/devbench.py --n 1024 --iters 2 > /dev/null 2>&1
