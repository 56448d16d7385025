OUT=gpurun_out/exp25; mkdir -p $OUT
for v in "$@"; do TFFFT_LIB=build/variants/$v/libtffft.so ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/l_$v.csv python tools/devbench.py --n 1024 --iters 2 > /dev/null 2>&1; done
for v in "$@"; do TFFFT_LIB=build/variants/$v/libtffft.so ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/f_$v.csv python tools/devbench.py --n 1024 --iters 2 --dtype float32 > /dev/null 2>&1; done
TFFFT_LIB=build/variants/direct/libtffft.so timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_direct.log 2>&1
