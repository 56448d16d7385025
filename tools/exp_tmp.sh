OUT=gpurun_out/exp45; mkdir -p $OUT
for m in 10 9; do TFFFT_TICKET_MINL=$m ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/l_$m.csv python tools/devbench.py --n 512 --iters 2 > /dev/null 2>&1; done
for m in 10 9; do TFFFT_TICKET_MINL=$m ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/f_$m.csv python tools/devbench.py --n 512 --iters 2 --dtype float32 > /dev/null 2>&1; done
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1
