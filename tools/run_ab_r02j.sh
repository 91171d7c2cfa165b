#!/bin/bash
# fp32 register kernel: packed f32x2 pairs vs scalar FFMA (device time, graph replay).
cd /root/repo; O=gpurun_out/ab_r02j.txt; : > $O
for i in 1 2; do for v in f32plain f32x2; do
  for a in "--config C2" "--n 7 --batch 1000000" "--n 16 --batch 1000000" "--n 24 --batch 1000000" "--n 30 --batch 1000000" "--n 32 --batch 1000000" "--n 30 --batch 100000" "--n 12 --batch 100000"; do
    python tools/fake_time.py fakebuild/librd_$v.so $a --dtype f32 --strategy thread --graph >> $O 2>&1; done
done; done
cat $O
