#!/bin/bash
# Run on the GPU box (under gpurun): plain bench, then the ncu launch list of
# the same command, then one full capture of the stage-3 column kernel.
set -x
OUT=gpurun_out/${1:-prof}
mkdir -p $OUT
CMD="python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1"
$CMD > $OUT/plain.json 2> $OUT/plain.err && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_list.log 2>&1
# stage-3 forward of the 5th pair (after the correctness pair + 3 warmups): col launches are
# 1b, 3, 3', 1b' per pair -> skip 4*4+1 col launches
$CMD > $OUT/plain2.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:col_fft -s 17 -c 1 \
    -o $OUT/stage3 $CMD > $OUT/ncu_full.log 2>&1
tail -2 $OUT/ncu_full.log
