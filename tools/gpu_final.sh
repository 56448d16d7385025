#!/bin/bash
# final check at HEAD: GPU suite and smoke (unless SKIP_TESTS=1), three default bench runs (box variance), the reference arm as the driver runs it
OUT=gpurun_out/${1:-final}; mkdir -p $OUT
if [ -z "$SKIP_TESTS" ]; then
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
fi
for i in 1 2 3; do
  s=$SECONDS
  timeout 600 python bench.py >> $OUT/bench3.json 2>> $OUT/bench3.err
  echo "bench run $i wall $((SECONDS - s)) s" >> $OUT/walls.txt
done
s=$SECONDS
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 3 > $OUT/bench_ref_k20.json 2> $OUT/bench_ref_k20.err
echo "reference arm K=20 W=3 wall $((SECONDS - s)) s" >> $OUT/walls.txt
