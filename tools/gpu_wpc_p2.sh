#!/bin/bash
# per-rank launch list of 1024^3 at p = 2 (local fabric) with and without the warp-per-column kernel
OUT=gpurun_out/${1:-wpcp2}
mkdir -p $OUT
for m in 0 2; do
  CMD="python -m paper_1406_5597_b200 bench --size 1024 --procs 2 --iters 3 --warmup 1"
  TFFFT_WPC=$m timeout 300 $CMD > $OUT/bench_1024_p2_wpc$m.csv 2>&1
  TFFFT_WPC=$m timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file $OUT/launches_1024_p2_wpc$m.csv $CMD > /dev/null 2>&1
done
