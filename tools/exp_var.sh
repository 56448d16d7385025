OUT=gpurun_out/exp3; mkdir -p $OUT
for v in "$@"; do echo "== $v"; TFFFT_LIB=build/variants/$v/libtffft.so timeout 300 python tools/devbench.py --n 1024 --iters 10 --check 2>&1 | tail -3; done > $OUT/ab.txt 2>&1
