#!/bin/bash
# THREAD stash kernel fp64 (W = 8): input prefetch distance x step-loop unroll.
cd /root/repo; O=gpurun_out/ab_pd.txt; : > $O
for rep in 1 2; do for v in $VARIANTS; do
  python tools/fake_time.py fakebuild/librd_$v.so --n 30 --batch 1000000 --graph >> $O 2>&1
  python tools/fake_time.py fakebuild/librd_$v.so --n 24 --batch 1000000 --graph >> $O 2>&1
done; done
cat $O
