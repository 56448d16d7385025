# A/B of row-kernel occupancy variants (built by tools/build_variants.sh)
mkdir -p gpurun_out/ab
for v in "$@"; do
  TFFFT_LIB=build/variants/$v/libtffft.so ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/ab/$v.csv python tools/devbench.py --n 1024 --iters 2 > /dev/null 2>&1
  echo "== $v"; python tools/launch_summary.py gpurun_out/ab/$v.csv 2>/dev/null | grep rows
  TFFFT_LIB=build/variants/$v/libtffft.so python tools/devbench.py --n 1024 --iters 10 2>&1 | tail -2
done
