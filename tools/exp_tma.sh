OUT=gpurun_out/exp13; mkdir -p $OUT
for cfg in "0 0" "1 0" "1 1"; do set -- $cfg
 echo "== TMA_COLS=$1 STORE=$2"; TFFFT_TMA_COLS=$1 TFFFT_TMA_STORE=$2 timeout 300 python tools/devbench.py --n 1024 --iters 10 --check 2>&1 | tail -3
 echo "== TMA_COLS=$1 STORE=$2 f32"; TFFFT_TMA_COLS=$1 TFFFT_TMA_STORE=$2 timeout 300 python tools/devbench.py --n 1024 --dtype float32 --iters 10 --check 2>&1 | tail -3
done > $OUT/ab.txt 2>&1
TFFFT_TMA_COLS=1 TFFFT_TMA_STORE=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/launches.csv python tools/devbench.py --n 1024 --iters 2 > /dev/null 2>&1
