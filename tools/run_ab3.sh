#!/bin/bash
# A/B of two variant libraries on the ID/FD configs + GPU suite on the second.
# usage: tools/run_ab3.sh OLD NEW   (fakebuild/librd_<v>.so)
cd /root/repo; mkdir -p gpurun_out
o=$1; nw=$2
for i in 1 2 3; do for v in $o $nw; do for a in "--config C3" "--config C3 --dtype f32" "--config C5" "--config C2" "--config C4 --fd" "--config C3 --batch 100000 --strategy reverse" "--n 100 --batch 100000 --strategy reverse"; do
  python tools/fake_time.py fakebuild/librd_$v.so $a; done; done; done > gpurun_out/ab3.txt 2>&1
cp fakebuild/librd_$nw.so paper_1609_04493_b200/librd.so
echo "== tests $nw: $(timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3)" >> gpurun_out/ab3.txt
cat gpurun_out/ab3.txt
