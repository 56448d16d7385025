#!/bin/bash
# A/B of library variants built by tools/build_variants.sh: launch lists (ncu) per variant
# usage (on the GPU box): bash tools/exp_var.sh <outdir> v1 v2 ...
OUT=gpurun_out/$1; shift; mkdir -p $OUT
for v in "$@"; do
  TFFFT_LIB=build/variants/$v/libtffft.so ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file $OUT/l_$v.csv python tools/devbench.py --n 1024 --iters 2 > /dev/null 2>&1
done
