#!/bin/bash
# fp32 n = 17..26: register kernel (prod) vs stash kernel (stash16); then the GPU suite on prod.
cd /root/repo; O=gpurun_out/ab_r02l.csv; echo "lib,n,B,ms" > $O
for v in stash16 prod; do for n in 17 18 19 20 21 22 23 24 25 26; do for B in 100000 1000000; do
  python tools/fake_time.py fakebuild/librd_$v.so --n $n --batch $B --dtype f32 --strategy thread --graph 2>&1 | awk -v v=$v -v n=$n -v B=$B '/ ms$/{print v","n","B","$(NF-1)}' >> $O
done; done; done
cat $O
echo "== tests: $(timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4)"
