#!/bin/bash
# full-prefetch TMA column kernel (TFFFT_TMA_FPF=1) vs default: correctness, pair times, launch lists
OUT=gpurun_out/${1:-fpf}
mkdir -p $OUT
TFFFT_TMA_FPF=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch.py -m gpu -q -x > $OUT/pytest_fpf.log 2>&1; echo "exit $?" >> $OUT/pytest_fpf.log
for rep in 1 2; do
for F in 0 1; do
  for dt in float64 float32; do
    echo "FPF=$F $dt" >> $OUT/devbench.txt
    TFFFT_TMA_FPF=$F timeout 300 python tools/devbench.py --n 1024 --iters 10 --dtype $dt >> $OUT/devbench.txt 2>&1
  done
done
done
CMD="python tools/devbench.py --n 1024 --iters 1"
for F in 0 1; do
  TFFFT_TMA_FPF=$F WARM=1 $CMD > /dev/null 2>&1 && TFFFT_TMA_FPF=$F WARM=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/launches_fpf$F.csv $CMD > /dev/null 2>&1
  echo "ncu $F $?" >> $OUT/devbench.txt
done
