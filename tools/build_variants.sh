#!/bin/bash
# build experimental variants of libtffft.so into build/variants/<name>/libtffft.so
set -e
cd "$(dirname "$0")/../paper_1406_5597_b200/csrc"
build() {
  name=$1; shift
  mkdir -p ../../build/variants/$name
  make -s clean >/dev/null
  make -s -j3 EXTRA_NVCC_FLAGS="$*" >/dev/null
  cp ../libtffft.so ../../build/variants/$name/libtffft.so
}
while [ $# -gt 0 ]; do build "$1" "$2"; shift 2; done
make -s clean >/dev/null; make -s -j3 >/dev/null
