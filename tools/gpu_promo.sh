#!/bin/bash
# L2 promotion of the stage-3 load maps: ncu launch lists + live pairs, one box
OUT=gpurun_out/${1:-promo}
mkdir -p $OUT
for w in 2 1; do
for pr in 0 3 2; do
  echo "== TFFFT_WPC=$w TFFFT_TMA_PROMO=$pr" >> $OUT/ab.txt
  TFFFT_WPC=$w TFFFT_TMA_PROMO=$pr timeout 300 python tools/devbench.py --n 1024 --iters 10 >> $OUT/ab.txt 2>&1
  TFFFT_WPC=$w TFFFT_TMA_PROMO=$pr timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
     --log-file $OUT/l_w${w}_p$pr.csv python tools/devbench.py --n 1024 --iters 1 > /dev/null 2>&1
done
done
