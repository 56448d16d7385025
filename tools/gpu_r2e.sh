#!/bin/bash
# p > 1 TMA column kernels: GPU suite + launch lists of 512^3 at p=1,2,4 and 1024^3 at p=1,2 (local fabric)
OUT=gpurun_out/${1:-r2e}
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
for cfg in "512 1" "512 2" "512 4" "1024 1" "1024 2"; do
  set -- $cfg
  CMD="python -m paper_1406_5597_b200 bench --size $1 --procs $2 --iters 3 --warmup 1"
  timeout 300 $CMD > $OUT/bench_$1_p$2.csv 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file $OUT/launches_$1_p$2.csv $CMD > /dev/null 2>&1
  echo "$cfg ncu $?" >> $OUT/status.txt
done
