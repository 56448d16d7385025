#!/bin/bash
# A/B of library builds on one box: exp_libs.sh OUT lib1 lib2 ...  ("default" = the in-tree library)
OUT=gpurun_out/$1; shift
mkdir -p $OUT
libpath() { [ "$1" = default ] && echo paper_1406_5597_b200/libtffft.so || echo build/variants/$1/libtffft.so; }
for v in "$@"; do
  TFFFT_LIB=$(libpath $v) timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_races.py -m gpu -q -x -k "tma or poison or 1024" > $OUT/pytest_$v.log 2>&1; echo "exit $?" >> $OUT/pytest_$v.log
done
for rep in 1 2; do
  for v in "$@"; do
    for dt in float64 float32; do
      echo "$v $dt" >> $OUT/devbench.txt
      TFFFT_LIB=$(libpath $v) timeout 300 python tools/devbench.py --n 1024 --iters 10 --dtype $dt >> $OUT/devbench.txt 2>&1
    done
  done
done
CMD="python tools/devbench.py --n 1024 --iters 1"
for v in "$@"; do
  TFFFT_LIB=$(libpath $v) WARM=1 $CMD > /dev/null 2>&1 && TFFFT_LIB=$(libpath $v) WARM=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/launches_$v.csv $CMD > /dev/null 2>&1
  echo "ncu $v $?" >> $OUT/devbench.txt
done
