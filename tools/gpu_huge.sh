#!/bin/bash
# A/B: plan buffers from torch's cudaMalloc (2 MB pages) vs 512 MB-aligned VMM mappings (tools/micro/hugealloc.cu)
OUT=gpurun_out/huge; mkdir -p $OUT
for rep in 1 2; do
  for h in "" 1; do
    echo "== HUGE_ALLOC=$h rep $rep" >> $OUT/live.txt
    HUGE_ALLOC=$h HUGE_VERBOSE=1 timeout 300 python tools/devbench.py --n 1024 --iters 20 --check >> $OUT/live.txt 2>&1
  done
done
for h in "" 1; do
  HUGE_ALLOC=$h timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $OUT/launches_huge$h.csv python tools/devbench.py --n 1024 --iters 3 > $OUT/ncu$h.log 2>&1
  echo "== HUGE_ALLOC=$h" >> $OUT/launches.txt
  python tools/launch_summary.py $OUT/launches_huge$h.csv >> $OUT/launches.txt 2>&1
done
for al in 2 32 64; do
  echo "== HUGE_ALLOC=1 HUGE_ALIGN_MB=$al" >> $OUT/live.txt
  HUGE_ALLOC=1 HUGE_ALIGN_MB=$al timeout 300 python tools/devbench.py --n 1024 --iters 20 >> $OUT/live.txt 2>&1
done
