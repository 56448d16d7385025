#!/bin/bash
# n2 = 2048 row kernels (BASELINE config 4's per-rank rows): radix schedule / occupancy variants, ncu launch lists
# usage: bash tools/gpu_rows10.sh <outdir> <variant> ...   (variants under build/variants; "base" = the in-tree library)
OUT=gpurun_out/${1:-rows10}; shift
mkdir -p $OUT
for v in "$@"; do
  LIB=build/variants/$v/libtffft.so
  [ $v = base ] && LIB=paper_1406_5597_b200/libtffft.so
  TFFFT_LIB=$LIB timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file $OUT/l_$v.csv python tools/devbench.py --shape 256,2048,2048 --iters 2 --check > $OUT/dev_$v.txt 2>&1
done
