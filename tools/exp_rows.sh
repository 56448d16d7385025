OUT=gpurun_out/exp19; mkdir -p $OUT
ncu --set full --import-source on --clock-control none -k regex:"r2c_rows|c2r_rows" -s 2 -c 2 -o $OUT/rows python tools/devbench.py --n 1024 --iters 1 > $OUT/ncu.log 2>&1
