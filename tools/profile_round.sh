#!/bin/bash
# Run on the GPU box (under gpurun): plain bench, then the ncu launch list of
# the same command, then one full capture of the stage-3 column kernel
# (selected through the library's NVTX ranges: forward call, stage 3).
set -x
OUT=gpurun_out/${1:-prof}
mkdir -p $OUT
CMD="python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1"
$CMD > $OUT/plain.json 2> $OUT/plain.err && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_list.log 2>&1
# stage-3 forward of the 5th forward call (correctness pair + 3 warm-ups first)
$CMD > $OUT/plain2.json 2>&1 && \
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "tffft.forward/stage3/" \
    -k regex:col_ -s 4 -c 1 -o $OUT/stage3 $CMD > $OUT/ncu_full.log 2>&1
tail -2 $OUT/ncu_full.log
