#!/bin/bash
# round-2 GPU session b: full GPU suite (incl. full-size parity), smoke, bench, CPU full pair
OUT=gpurun_out/${1:-r2b}
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 900 python tools/cpu_full_pair.py --grid 1024 --out $OUT/cpu_full_pair.json > $OUT/cpu_full_pair.log 2>&1
