#!/bin/bash
# Register ID kernel: inputs loaded PD links ahead inside the forward sweep vs all up front.
cd /root/repo; O=gpurun_out/ab_lazy.txt; : > $O
for rep in 1 2; do for v in base lazy4 lazy8; do
  for n in 24 30 32; do python tools/fake_time.py fakebuild/librd_$v.so --n $n --batch 1000000 --dtype f32 --graph >> $O 2>&1; done
  python tools/fake_time.py fakebuild/librd_$v.so --config C2 --dtype f32 --graph >> $O 2>&1
  for n in 7 12; do python tools/fake_time.py fakebuild/librd_$v.so --n $n --batch 1000000 --dtype f64 --graph >> $O 2>&1; done
  python tools/fake_time.py fakebuild/librd_$v.so --config C2 --dtype f64 --graph >> $O 2>&1
done; done
cat $O
