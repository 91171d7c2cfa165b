#!/bin/bash
# fp64 register kernel (with re-derived sin/cos) for 13 <= n <= 16 vs the stash kernel.
cd /root/repo; O=gpurun_out/ab_r02p.csv; echo "lib,n,B,ms" > $O
for v in prod f64max16; do for n in 13 14 15 16; do for B in 20000 100000 1000000; do
  python tools/fake_time.py fakebuild/librd_$v.so --n $n --batch $B --dtype f64 --strategy thread --graph 2>&1 | awk -v v=$v -v n=$n -v B=$B '/ ms$/{print v","n","B","$(NF-1)}' >> $O
done; done; done
cat $O
