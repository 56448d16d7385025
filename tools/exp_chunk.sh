OUT=gpurun_out/exp1; mkdir -p $OUT
for K in 0 2 4 8 16; do for D in 1 2; do
  [ $K = 0 ] && [ $D = 2 ] && continue
  echo "== K=$K D=$D"; TFFFT_S1_CHUNK=$K TFFFT_S1_DEPTH=$D timeout 300 python tools/devbench.py --n 1024 --iters 10 --check 2>&1 | tail -3
done; done > $OUT/chunk.txt 2>&1
TFFFT_S1_CHUNK=4 timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_chunk.log 2>&1
