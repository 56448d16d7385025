#!/bin/bash
# live (power-capped) A/B of library variants: alternating devbench pairs, 1024^3 f64
# usage (on the GPU box): bash tools/exp_live.sh <outdir> v1 v2 ...
OUT=gpurun_out/$1; shift; mkdir -p $OUT
for rep in 1 2 3; do for v in "$@"; do
  echo "== $v rep$rep"; TFFFT_LIB=build/variants/$v/libtffft.so timeout 120 python tools/devbench.py --n 1024 --iters 30 2>&1 | tail -2
done; done > $OUT/devbench.txt 2>&1
