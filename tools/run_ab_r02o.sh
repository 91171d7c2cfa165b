#!/bin/bash
# fp64 register kernel with the recomputing backward sweep: at any batch (p9any) and from n = 6 (p6any)
# vs the product (p9: n = 9..12 only up to 300k states); then the GPU suite on p9.
cd /root/repo; O=gpurun_out/ab_r02o.csv; echo "lib,n,B,ms" > $O
for v in p9 p9any p6any; do
  for n in 6 7 8 9 10 11 12; do for B in 100000 1000000; do
    python tools/fake_time.py fakebuild/librd_$v.so --n $n --batch $B --dtype f64 --strategy thread --graph 2>&1 | awk -v v=$v -v n=$n -v B=$B '/ ms$/{print v","n","B","$(NF-1)}' >> $O
  done; done
done
cat $O
echo "== tests: $(timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3)"
