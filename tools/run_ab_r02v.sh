#!/bin/bash
# Register ABA for longer chains (fp64 13..16, fp32 13..24) vs the workspace kernel.
cd /root/repo; O=gpurun_out/ab_r02v.csv; echo "lib,dtype,n,B,ms" > $O
for v in noabas abaw; do
  for n in 13 14 16; do for B in 100000 1000000; do
    python tools/fake_time.py fakebuild/librd_$v.so --n $n --batch $B --dtype f64 --fd --graph 2>&1 | awk -v v=$v -v n=$n -v B=$B '/ ms$/{print v",f64,"n","B","$(NF-1)}' >> $O
  done; done
  for n in 13 16 18 20 22 24; do for B in 100000 1000000; do
    python tools/fake_time.py fakebuild/librd_$v.so --n $n --batch $B --dtype f32 --fd --graph 2>&1 | awk -v v=$v -v n=$n -v B=$B '/ ms$/{print v",f32,"n","B","$(NF-1)}' >> $O
  done; done
done
cat $O
