#!/bin/bash
# fp32 register kernel, packed (pk1) vs scalar (pk0), every n = 1..32 at 1e5 and 1e6 states.
cd /root/repo; O=gpurun_out/ab_r02k.csv; echo "lib,n,B,ms" > $O
for v in pk0 pk1; do
  for n in $(seq 1 32); do for B in 100000 1000000; do
    python tools/fake_time.py fakebuild/librd_$v.so --n $n --batch $B --dtype f32 --strategy thread --graph 2>&1 | awk -v v=$v -v n=$n -v B=$B '/ ms$/{print v","n","B","$(NF-1)}' >> $O
  done; done
done
cat $O
