#!/bin/bash
# full ncu captures of the n2 = 1024 row kernels (1024^3 float64)
OUT=gpurun_out/${1:-rowsfull}
mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:c2r_rows -s 1 -c 1 -o $OUT/c2r \
    python tools/devbench.py --n 1024 --iters 1 > $OUT/ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:r2c_rows -s 1 -c 1 -o $OUT/r2c \
    python tools/devbench.py --n 1024 --iters 1 > $OUT/ncu2.log 2>&1
