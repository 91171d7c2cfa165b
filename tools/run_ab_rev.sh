#!/bin/bash
cd /root/repo; mkdir -p gpurun_out/r02
out=gpurun_out/r02/ab_rev.txt; : > $out
for rep in 1 2; do
for so in base rev_4_2 rev_2_2 rev_mb3 rev_8_4_mb3; do
  python tools/fake_time.py fakebuild/$so.so --config C4 --batch 1000000 --strategy reverse >> $out 2>&1
  python tools/fake_time.py fakebuild/$so.so --config C4 --batch 100000 --strategy reverse >> $out 2>&1
  python tools/fake_time.py fakebuild/$so.so --config C3 --batch 65536 --strategy reverse >> $out 2>&1
done; done
