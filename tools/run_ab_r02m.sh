#!/bin/bash
# Balanced launch geometry (every thread the same number of states) for ABA and REVERSE.
cd /root/repo; O=gpurun_out/ab_r02m.txt; : > $O
for i in 1 2; do for v in head bal; do
  for a in "--config C4 --fd" "--config C4 --fd --dtype f32" "--n 30 --batch 100000 --fd" "--n 200 --batch 20000 --fd" "--n 10 --batch 1000000 --fd" "--n 100 --batch 150000 --fd"; do
    python tools/fake_time.py fakebuild/librd_$v.so $a --graph >> $O 2>&1; done
  for a in "--n 100 --batch 100000" "--n 100 --batch 1000000" "--n 30 --batch 16384" "--n 30 --batch 65536" "--n 200 --batch 100000" "--n 64 --batch 300000"; do
    python tools/fake_time.py fakebuild/librd_$v.so $a --strategy reverse --graph >> $O 2>&1; done
done; done
cat $O
