#!/bin/bash
# generic env A/B on one box: exp_ab.sh OUT VAR "vals" [devbench args]
OUT=gpurun_out/$1; VAR=$2; VALS=$3; shift 3
mkdir -p $OUT
for v in $VALS; do
  env $VAR=$v timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_races.py tests/test_gpu_fullsize.py -m gpu -q -x -k "tma or poison or 1024_cubed" > $OUT/pytest_$v.log 2>&1; echo "exit $?" >> $OUT/pytest_$v.log
done
for rep in 1 2; do
  for v in $VALS; do
    for dt in float64 float32; do
      echo "$VAR=$v $dt" >> $OUT/devbench.txt
      env $VAR=$v timeout 300 python tools/devbench.py --n 1024 --iters 10 --dtype $dt "$@" >> $OUT/devbench.txt 2>&1
    done
  done
done
CMD="python tools/devbench.py --n 1024 --iters 1 $*"
for v in $VALS; do
  env $VAR=$v WARM=1 $CMD > /dev/null 2>&1 && env $VAR=$v WARM=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/launches_$v.csv $CMD > /dev/null 2>&1
  echo "ncu $v $?" >> $OUT/devbench.txt
done
