OUT=gpurun_out/exp14; mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -x -q -k "tma_column" > $OUT/pytest_tma.log 2>&1
timeout 300 tools/micro/l2_bw > $OUT/l2_bw.txt 2>&1
