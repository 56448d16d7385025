# devbench A/B of library variants built by tools/build_variants.sh: ab_var.sh <n> <dtype> v1 v2 ...
n=$1; dt=$2; shift 2
for v in "$@"; do
  echo "== $v"; TFFFT_LIB=build/variants/$v/libtffft.so python tools/devbench.py --n $n --dtype $dt --iters 10 --check 2>&1 | tail -3
done
