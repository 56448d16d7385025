OUT=gpurun_out/exp26; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/l64.csv python tools/devbench.py --n 1024 --iters 2 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/l32.csv python tools/devbench.py --n 1024 --iters 2 --dtype float32 > /dev/null 2>&1
