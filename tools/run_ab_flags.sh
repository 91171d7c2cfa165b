#!/bin/bash
# fp32 register kernel (n = 30): ptxas option variants of its translation unit.
cd /root/repo; O=gpurun_out/ab_flags.txt; : > $O
for rep in 1 2; do for v in base fl1 fl2 fl3 fl4; do
  for n in 28 30 32; do python tools/fake_time.py fakebuild/librd_$v.so --n $n --batch 1000000 --dtype f32 --graph >> $O 2>&1; done
done; done
cat $O
