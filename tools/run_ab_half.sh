#!/bin/bash
# THREAD stash kernel: two 4-warp CTAs per SM (half the TMEM / shared memory each) vs one 8-warp CTA.
cd /root/repo; O=gpurun_out/ab_half.txt; : > $O
python tools/ws_check.py fakebuild/librd_half.so --n 17,22,30 --batch 1000,70001,1000000 --time-n 30 >> $O 2>&1
for rep in 1 2; do for v in base half; do
  for B in 100000 1000000 2000000 10000000; do python tools/fake_time.py fakebuild/librd_$v.so --n 30 --batch $B --graph >> $O 2>&1; done
  python tools/fake_time.py fakebuild/librd_$v.so --n 20 --batch 1000000 --graph >> $O 2>&1
  python tools/fake_time.py fakebuild/librd_$v.so --n 24 --batch 1000000 --graph >> $O 2>&1
done; done
cat $O
