OUT=gpurun_out/exp16; mkdir -p $OUT
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/f32.csv python tools/devbench.py --n 1024 --dtype float32 --iters 2 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/f64_512.csv python tools/devbench.py --n 512 --iters 2 > /dev/null 2>&1
