OUT=gpurun_out/pw; mkdir -p $OUT
nvidia-smi -q -d POWER,CLOCK,PERFORMANCE > $OUT/smi_q.txt 2>&1
nvidia-smi --query-gpu=timestamp,power.draw,power.limit,enforced.power.limit,clocks.sm,clocks.mem,clocks_event_reasons.active --format=csv -lms 50 > $OUT/trace.csv 2>&1 &
P=$!
python tools/devbench.py --n 1024 --iters 60 > $OUT/devbench.txt 2>&1
kill $P
