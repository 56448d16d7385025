OUT=gpurun_out/exp9; mkdir -p $OUT
TFFFT_WS=1 TFFFT_WS_EF=0 ncu --set full --import-source on --clock-control none -k regex:col_ws -s 4 -c 2 -o $OUT/ws python tools/devbench.py --n 1024 --iters 1 > $OUT/ncu.log 2>&1
