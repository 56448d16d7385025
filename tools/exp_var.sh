OUT=gpurun_out/exp18; mkdir -p $OUT
for v in "$@"; do echo "== $v"; TFFFT_LIB=build/variants/$v/libtffft.so timeout 300 python tools/devbench.py --n 1024 --dtype float32 --iters 10 --check 2>&1 | tail -3; done > $OUT/ab.txt 2>&1
for v in "$@"; do TFFFT_LIB=build/variants/$v/libtffft.so ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/l_$v.csv python tools/devbench.py --n 1024 --dtype float32 --iters 2 > /dev/null 2>&1; done
TFFFT_LIB=build/variants/f2cta/libtffft.so timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_widen.log 2>&1
