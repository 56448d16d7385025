#!/bin/bash
# same-box A/B of TFFFT_WPC modes (0 off, 1 all passes, 2 stage-1b passes only), interleaved
OUT=gpurun_out/${1:-wpcab}
mkdir -p $OUT
for rep in 1 2 3; do
for m in 0 2 1; do
  echo "== TFFFT_WPC=$m f64 rep $rep" >> $OUT/ab.txt
  TFFFT_WPC=$m timeout 300 python tools/devbench.py --n 1024 --iters 20 >> $OUT/ab.txt 2>&1
done
done
for m in 0 1; do
  echo "== TFFFT_WPC=$m f32" >> $OUT/ab.txt
  TFFFT_WPC=$m timeout 300 python tools/devbench.py --n 1024 --dtype float32 --iters 20 >> $OUT/ab.txt 2>&1
done
