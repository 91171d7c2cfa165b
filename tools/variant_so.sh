#!/bin/bash
# Build a variant librd.so with extra nvcc defines for ONE source file (A/B timing).
# usage: tools/variant_so.sh <source.cu basename> <out.so> [-DFOO=1 ...]
set -e
cd "$(dirname "$0")/.."
src=$1; out=$2; shift 2
python -m paper_1609_04493_b200._build >/dev/null
mkdir -p fakebuild/obj
objs=()
for o in build/rd/*.o; do
  if [ "$(basename $o)" = "$src.o" ]; then
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2,-Wall,-Wshadow \
      -Iinclude -Ipaper_1609_04493_b200/csrc "$@" -c paper_1609_04493_b200/csrc/$src -o fakebuild/obj/$src.o
    objs+=(fakebuild/obj/$src.o)
  else
    objs+=($o)
  fi
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$out" "${objs[@]}"
echo "$out"
