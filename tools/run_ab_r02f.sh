#!/bin/bash
# REVERSE: register prefetch (cur) vs cp.async ring depths; device time (graph replay).
cd /root/repo; O=gpurun_out/ab_r02f.txt; : > $O
for i in 1 2; do for v in cur revring5 revring8 revring12; do
  for a in "--n 100 --batch 1000000" "--n 100 --batch 100000" "--n 30 --batch 16384" "--n 30 --batch 1000000" "--n 200 --batch 100000" "--n 100 --batch 1000000 --dtype f32"; do
    python tools/fake_time.py fakebuild/librd_$v.so $a --strategy reverse --graph >> $O 2>&1; done
done; done
cat $O
echo "== tests: $(timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4)" >> $O; tail -5 $O
