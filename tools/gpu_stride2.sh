#!/bin/bash
# stage 3 at the 1 MB row stride of a p = 8 rank: col_tma_kernel (TFFFT_WPC=2) against col_wpc_kernel (TFFFT_WPC=1)
OUT=gpurun_out/${1:-stride2}
mkdir -p $OUT
for m in 2 1; do
  for n1 in 128 256; do
  TFFFT_WPC=$m timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file $OUT/l_${n1}_wpc$m.csv python tools/devbench.py --shape 1024,$n1,1024 --iters 3 > $OUT/dev_${n1}_wpc$m.txt 2>&1
  done
  CMD="python -m paper_1406_5597_b200 bench --size 1024 --procs 8 --iters 2 --warmup 1"
  TFFFT_WPC=$m timeout 600 $CMD > $OUT/bench_p8_wpc$m.csv 2>&1
  TFFFT_WPC=$m timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file $OUT/l_p8_wpc$m.csv $CMD > /dev/null 2>&1
done
