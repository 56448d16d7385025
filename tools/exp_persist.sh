#!/bin/bash
# plane-chunked stage 1 with a persisting-L2 window over each chunk (TFFFT_S1_PERSIST)
OUT=gpurun_out/${1:-per}
mkdir -p $OUT
TFFFT_S1_CHUNK=4 TFFFT_S1_PERSIST=1 timeout 600 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -k "1024_cubed_p1_vs_oracle and float64" > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
for rep in 1 2; do
for cfg in "0 0" "4 1" "8 1" "2 1" "4 0"; do
  set -- $cfg
  echo "CHUNK=$1 PERSIST=$2" >> $OUT/devbench.txt
  TFFFT_S1_CHUNK=$1 TFFFT_S1_PERSIST=$2 timeout 300 python tools/devbench.py --n 1024 --iters 10 >> $OUT/devbench.txt 2>&1
done
done
CMD="python tools/devbench.py --n 1024 --iters 1"
TFFFT_S1_CHUNK=4 TFFFT_S1_PERSIST=1 WARM=1 $CMD > /dev/null 2>&1 && TFFFT_S1_CHUNK=4 TFFFT_S1_PERSIST=1 WARM=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --cache-control none --csv --log-file $OUT/launches_k4p.csv $CMD > /dev/null 2>&1
echo "ncu $?" >> $OUT/devbench.txt
