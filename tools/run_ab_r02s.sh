#!/bin/bash
# fp64 register kernel, capped builds at every batch: 3 vs 4 resident CTAs per SM (prod: uncapped below 300k).
cd /root/repo; O=gpurun_out/ab_r02s.csv; echo "lib,n,B,ms" > $O
for v in prod cap3 cap4; do for n in 6 7 8 9 10 12; do for B in 100000 1000000; do
  python tools/fake_time.py fakebuild/librd_$v.so --n $n --batch $B --strategy thread --graph 2>&1 | awk -v v=$v -v n=$n -v B=$B '/ ms$/{print v","n","B","$(NF-1)}' >> $O
done; done; done
cat $O
