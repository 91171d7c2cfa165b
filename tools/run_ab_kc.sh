#!/bin/bash
# THREAD stash kernel fp64: link constants as LDG.128 pairs from an L1-resident global table vs constant-bank LDC.
cd /root/repo; O=gpurun_out/ab_kc.txt; : > $O
python tools/ws_check.py fakebuild/librd_kc.so --n 17,22,30 --batch 1000,70001,1000000 --time-n 30 >> $O 2>&1
for rep in 1 2; do for v in base kc; do
  for n in 20 24 30; do python tools/fake_time.py fakebuild/librd_$v.so --n $n --batch 1000000 --graph >> $O 2>&1; done
  python tools/fake_time.py fakebuild/librd_$v.so --n 30 --batch 10000000 --graph >> $O 2>&1
done; done
cat $O
