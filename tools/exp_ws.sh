OUT=gpurun_out/exp8; mkdir -p $OUT
for cfg in "0 1" "1 1" "1 0"; do set -- $cfg
 echo "== WS=$1 EF=$2"; TFFFT_WS=$1 TFFFT_WS_EF=$2 timeout 300 python tools/devbench.py --n 1024 --iters 10 --check 2>&1 | tail -3
done > $OUT/ab.txt 2>&1
echo "== f32" >> $OUT/ab.txt; TFFFT_WS=1 timeout 300 python tools/devbench.py --n 1024 --iters 10 --dtype float32 --check >> $OUT/ab.txt 2>&1
TFFFT_WS=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/launches.csv python tools/devbench.py --n 1024 --iters 2 > /dev/null 2>&1
TFFFT_WS=1 timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1
