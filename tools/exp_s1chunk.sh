#!/bin/bash
# plane-interleaved stage 1 experiment (TFFFT_S1_CHUNK planes per r2c+columns chunk) at 1024^3 f64
OUT=gpurun_out/${1:-s1c}
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tma_column" > $OUT/pytest_tma.log 2>&1; echo "exit $?" >> $OUT/pytest_tma.log
for K in 0 4 8 16 32 0; do
  echo "K=$K" >> $OUT/devbench.txt
  TFFFT_S1_CHUNK=$K timeout 300 python tools/devbench.py --n 1024 --iters 10 >> $OUT/devbench.txt 2>&1
done
CMD="python tools/devbench.py --n 1024 --iters 1"
TFFFT_S1_CHUNK=8 WARM=1 $CMD > /dev/null 2>&1 && TFFFT_S1_CHUNK=8 WARM=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --csv --log-file $OUT/launches_k8.csv $CMD > /dev/null 2>&1
echo "ncu $?" >> $OUT/devbench.txt
