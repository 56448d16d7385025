#!/bin/bash
OUT=gpurun_out/${1:-wpc2l}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_races.py -m gpu -x -q -k "wpc or poisoned or tma_column" > $OUT/pytest.log 2>&1; echo "pytest exit $?" >> $OUT/pytest.log
