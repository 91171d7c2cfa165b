#!/bin/bash
# fp32 A/B (OLD NEW) on C3 / C2 / n = 20 + GPU suite on NEW.
cd /root/repo; mkdir -p gpurun_out
o=$1; nw=$2
for i in 1 2 3; do for v in $o $nw; do for a in "--config C3 --dtype f32" "--config C2 --dtype f32" "--n 20 --batch 1000000 --dtype f32" "--config C3"; do
  python tools/fake_time.py fakebuild/librd_$v.so $a; done; done; done > gpurun_out/ab_f32.txt 2>&1
cp fakebuild/librd_$nw.so paper_1609_04493_b200/librd.so
echo "== tests $nw: $(timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3)" >> gpurun_out/ab_f32.txt
cat gpurun_out/ab_f32.txt
