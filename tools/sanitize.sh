#!/bin/bash
# one compute-sanitizer tool per gpurun call (B200_PROFILING.md): memcheck | racecheck | synccheck
TOOL=${1:-memcheck}
OUT=gpurun_out/san
mkdir -p $OUT
python tools/sanitize_cases.py > $OUT/plain_$TOOL.log 2>&1 && \
timeout 1500 compute-sanitizer --tool $TOOL --target-processes all --print-limit 50 \
    python tools/sanitize_cases.py > $OUT/$TOOL.log 2>&1
echo "exit $?" >> $OUT/$TOOL.log
