#!/bin/bash
# Build a variant librd.so with extra nvcc flags for SEVERAL source files (A/B timing).
# usage: tools/variant_multi.sh <out.so> "<flags>" <source.cu> [<source.cu> ...]
set -e
cd "$(dirname "$0")/.."
out=$1; flags=$2; shift 2
python -m paper_1609_04493_b200._build >/dev/null
mkdir -p fakebuild/obj
tag=$(basename $out .so)
objs=()
for o in build/rd/*.o; do
  src=$(basename $o .o)
  hit=0; for s in "$@"; do [ "$s" = "$src" ] && hit=1; done
  if [ $hit = 1 ]; then
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 $flags \
      -Iinclude -Ipaper_1609_04493_b200/csrc -c paper_1609_04493_b200/csrc/$src -o fakebuild/obj/$src.$tag.o &
    objs+=(fakebuild/obj/$src.$tag.o)
  else
    objs+=($o)
  fi
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$out" "${objs[@]}"
echo "$out"
