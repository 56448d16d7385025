#!/bin/bash
# n2 = 1024 row kernels: occupancy variants (1024^3 float64), ncu launch lists
OUT=gpurun_out/${1:-rows9}; shift
mkdir -p $OUT
for v in "$@"; do
  LIB=build/variants/$v/libtffft.so
  [ $v = base ] && LIB=paper_1406_5597_b200/libtffft.so
  TFFFT_LIB=$LIB timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file $OUT/l_$v.csv python tools/devbench.py --n 1024 --iters 2 > $OUT/dev_$v.txt 2>&1
done
