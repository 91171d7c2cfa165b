#!/bin/bash
# A/B: fp32 dh_link sin/cos as one FFMA2 polynomial pair (register kernel n > 8, REVERSE fp32).
cd /root/repo; O=gpurun_out/ab_sc2.txt; : > $O
for rep in 1 2; do for v in base sc2; do
  for n in 12 20 30; do
    python tools/fake_time.py fakebuild/librd_$v.so --n $n --batch 1000000 --dtype f32 --graph >> $O 2>&1
  done
  python tools/fake_time.py fakebuild/librd_$v.so --n 100 --batch 1000000 --dtype f32 --strategy reverse --graph >> $O 2>&1
done; done
cat $O
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/ab_sc2_pytest.txt 2>&1; tail -3 gpurun_out/ab_sc2_pytest.txt
