#!/bin/bash
# Build a variant librd.so with ONE source file edited by sed expressions (A/B timing).
# usage: tools/variant_src.sh <source.cu basename> <out.so> <sed-expr> [<sed-expr> ...]
set -e
cd "$(dirname "$0")/.."
src=$1; out=$2; shift 2
python -m paper_1609_04493_b200._build >/dev/null
mkdir -p fakebuild/src fakebuild/obj
cp paper_1609_04493_b200/csrc/$src fakebuild/src/$src
for e in "$@"; do sed -i "$e" fakebuild/src/$src; done
if cmp -s paper_1609_04493_b200/csrc/$src fakebuild/src/$src; then echo "variant_src: sed changed nothing" >&2; exit 1; fi
objs=()
for o in build/rd/*.o; do
  if [ "$(basename $o)" = "$src.o" ]; then
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 \
      -Iinclude -Ipaper_1609_04493_b200/csrc -c fakebuild/src/$src -o fakebuild/obj/$src.$(basename $out).o
    objs+=(fakebuild/obj/$src.$(basename $out).o)
  else
    objs+=($o)
  fi
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$out" "${objs[@]}"
echo "$out"
