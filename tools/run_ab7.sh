#!/bin/bash
# A/B OLD NEW on C3 f64 / f32, C2, n = 15 + GPU suite on NEW
cd /root/repo; mkdir -p gpurun_out
o=$1; nw=$2
for i in 1 2 3; do for v in $o $nw; do for a in "--config C3" "--config C3 --dtype f32" "--config C2" "--n 15 --batch 1000000" "--config C5"; do
  python tools/fake_time.py fakebuild/librd_$v.so $a; done; done; done > gpurun_out/ab7.txt 2>&1
cp fakebuild/librd_$nw.so paper_1609_04493_b200/librd.so
echo "== tests $nw: $(timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1)" >> gpurun_out/ab7.txt
cat gpurun_out/ab7.txt
