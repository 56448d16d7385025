for v in s1 s0; do for d in float64 float32; do
  echo "== $v $d"; TFFFT_LIB=build/variants/$v/libtffft.so python tools/devbench.py --n 1024 --dtype $d --iters 10 --check 2>&1 | tail -3
done; done
