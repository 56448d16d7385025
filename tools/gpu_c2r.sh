#!/bin/bash
OUT=gpurun_out/${1:-c2r}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "forward_inverse_vs_oracle or known_answers or non_hermitian" > $OUT/pytest.log 2>&1; echo "pytest exit $?" >> $OUT/pytest.log
grep -q "pytest exit 0" $OUT/pytest.log || exit 1
for sh in 1024,1024,1024 512,512,512 256,2048,2048; do
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file $OUT/l_$(echo $sh | tr ',' 'x').csv python tools/devbench.py --shape $sh --iters 2 --check > $OUT/dev_$(echo $sh | tr ',' 'x').txt 2>&1
done
for rep in 1 2; do timeout 300 python tools/devbench.py --n 1024 --iters 20 >> $OUT/live.txt 2>&1; done
