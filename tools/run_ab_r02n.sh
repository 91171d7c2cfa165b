#!/bin/bash
# Register kernel: backward sweep re-deriving sin/cos (rc: fp32 n >= 17, fp64 n >= 9) vs keeping them (norc).
cd /root/repo; O=gpurun_out/ab_r02n.csv; echo "lib,dtype,n,B,ms" > $O
for v in norc rc; do
  for n in 17 20 24 25 26 27 28 30 32; do for B in 100000 1000000; do
    python tools/fake_time.py fakebuild/librd_$v.so --n $n --batch $B --dtype f32 --strategy thread --graph 2>&1 | awk -v v=$v -v n=$n -v B=$B '/ ms$/{print v",f32,"n","B","$(NF-1)}' >> $O
  done; done
  for n in 9 10 11 12; do for B in 100000 262144; do
    python tools/fake_time.py fakebuild/librd_$v.so --n $n --batch $B --dtype f64 --strategy thread --graph 2>&1 | awk -v v=$v -v n=$n -v B=$B '/ ms$/{print v",f64,"n","B","$(NF-1)}' >> $O
  done; done
done
cat $O
