#!/bin/bash
# Build kernel-tuning variants of librpq.so into build/variants/ (development aid).
# usage: scripts/build_variants.sh "-DRPQ_LEVEL_MINB=2 -DRPQ_SLOTS=8" name ...
set -e
cd "$(dirname "$0")/.."
mkdir -p build/variants
while [ $# -ge 2 ]; do
  flags="$1"; name="$2"; shift 2
  d=build/variants/$name; mkdir -p $d
  for f in eval.cu graph.cu crpq.cu capi.cpp regex.cpp plan.cpp; do
    nvcc $flags -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 -Iinclude -Ipaper_2602_20748_b200/csrc --expt-relaxed-constexpr -c paper_2602_20748_b200/csrc/$f -o $d/$f.o &
  done
  wait
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/variants/librpq_$name.so $d/*.o -lcudart_static -lrt -ldl -lpthread
done
