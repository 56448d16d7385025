#!/bin/bash
# full GPU suite + bench lines + profiling round (launch list + one full stage-3 capture)
OUT=gpurun_out/${1:-r2f}
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err
for extra in "--dtype float32" "--grid 512" "--config turbulence --steps 5"; do
  timeout 600 python bench.py --no-cpu $extra >> $OUT/bench_lines.json 2>> $OUT/bench_lines.err
done
timeout 900 bash tools/profile_round.sh ${1:-r2f}/prof
