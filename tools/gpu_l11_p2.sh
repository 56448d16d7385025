#!/bin/bash
# 2048-point two-level column passes at the per-rank size of 2048^3 / 8 (8.6 GB real slab per rank), p = 2 on the local fabric
OUT=gpurun_out/${1:-l11p2}
mkdir -p $OUT
for sz in 512,2048,2048 2048,512,2048; do
  tag=$(echo $sz | tr ',' 'x')
  CMD="python -m paper_1406_5597_b200 bench --size $sz --procs 2 --iters 2 --warmup 1"
  timeout 600 $CMD > $OUT/bench_$tag.csv 2>&1
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file $OUT/launches_$tag.csv $CMD > /dev/null 2>&1
done
