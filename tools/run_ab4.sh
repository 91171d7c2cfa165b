#!/bin/bash
# Knob A/B: thread variants on C3 f64, ABA variants on C4 (median of 50, 3 rounds).
cd /root/repo; mkdir -p gpurun_out
for i in 1 2 3; do
  for v in cur t1 t2 t3 t4; do python tools/fake_time.py fakebuild/librd_$v.so --config C3; done
  for v in cur a1 a2 a3 a4; do python tools/fake_time.py fakebuild/librd_$v.so --config C4 --fd; done
done > gpurun_out/ab4.txt 2>&1
cat gpurun_out/ab4.txt
