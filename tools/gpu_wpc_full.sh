#!/bin/bash
# one full ncu capture of the warp-per-column stage-1b kernel (1024^3 float64) and of the wide variant
OUT=gpurun_out/${1:-wpcfull}
mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:col_wpc_kernel -s 2 -c 1 -o $OUT/wpc_s1b \
    python tools/devbench.py --n 1024 --iters 1 > $OUT/ncu1.log 2>&1
TFFFT_WPC=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:col_wpc_kernel -s 5 -c 1 -o $OUT/wpc_s3 \
    python tools/devbench.py --n 1024 --iters 1 > $OUT/ncu2.log 2>&1
