#!/bin/bash
OUT=gpurun_out/${1:-wpc4}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_races.py -m gpu -x -q -k "wpc or poisoned" > $OUT/pytest.log 2>&1; echo "pytest exit $?" >> $OUT/pytest.log
grep -q "pytest exit 0" $OUT/pytest.log || exit 1
for rep in 1 2; do
for m in 2 1; do
  echo "== TFFFT_WPC=$m f64 rep $rep" >> $OUT/ab.txt
  TFFFT_WPC=$m timeout 300 python tools/devbench.py --n 1024 --iters 20 >> $OUT/ab.txt 2>&1
done
done
for m in 2 1; do
TFFFT_WPC=$m timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file $OUT/launches_wpc$m.csv python tools/devbench.py --n 1024 --iters 2 > /dev/null 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file $OUT/launches_512.csv python tools/devbench.py --n 512 --iters 2 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file $OUT/launches_f32.csv python tools/devbench.py --n 1024 --dtype float32 --iters 2 > /dev/null 2>&1
