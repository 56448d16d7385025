#!/bin/bash
# One GPU-box session: gpu tests, the bench lines, then the profiling round.
OUT=gpurun_out/${1:-r}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
for extra in "--dtype float32" "--grid 512" "--config turbulence --steps 5"; do
  timeout 600 python bench.py --no-cpu $extra >> $OUT/bench_lines.json 2>> $OUT/bench_lines.err
done
timeout 900 bash tools/profile_round.sh ${1:-r}/prof
for extra in "--dtype float32" "--grid 512"; do
  tag=$(echo $extra | tr -d ' -')
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/${1:-r}/prof/launches_$tag.csv python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 $extra > /dev/null 2>&1
done
