#!/bin/bash
# A/B of the column-kernel store flavour (TFFFT_COL_STORE 0/1/2): devbench pair times (alternating), then ncu launch lists
OUT=gpurun_out/${1:-st}; mkdir -p $OUT
for rep in 1 2; do for v in st0 st1 st2; do for dt in float64 float32; do
  echo "== $v $dt rep$rep"; TFFFT_LIB=build/variants/$v/libtffft.so timeout 120 python tools/devbench.py --n 1024 --dtype $dt --iters 10 --check 2>&1 | tail -3
done; done; done > $OUT/devbench.txt 2>&1
bash tools/exp_var.sh ${1:-st} st0 st1 st2
