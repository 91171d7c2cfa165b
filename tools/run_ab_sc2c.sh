#!/bin/bash
# fp32 paired sin/cos in the other dh_link users: register ABA (n <= 20), CHUNK, prismatic ABA; and the
# per-length register ID rule.
cd /root/repo; O=gpurun_out/ab_sc2c.txt; : > $O
for v in base sc2c; do
  for n in 7 12 16 20; do python tools/fake_time.py fakebuild/librd_$v.so --n $n --batch 1000000 --fd --dtype f32 --graph >> $O 2>&1; done
  python tools/fake_time.py fakebuild/librd_$v.so --n 100 --batch 10000 --strategy chunk:8 --dtype f32 --graph >> $O 2>&1
  for n in 12 19 30; do python tools/fake_time.py fakebuild/librd_$v.so --n $n --batch 1000000 --dtype f32 --graph >> $O 2>&1; done
done
cat $O
