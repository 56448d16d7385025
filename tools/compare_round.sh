# the paper's A/B (STRIDED vs TRANSPOSE) on one B200 with the current kernels
OUT=gpurun_out/${1:-cmp}; mkdir -p $OUT
{ python -m paper_1406_5597_b200 compare --size 512 --procs 1,2,4 --iters 5
  python -m paper_1406_5597_b200 compare --size 1024 --procs 1 --iters 3; } > $OUT/compare.txt 2>&1
