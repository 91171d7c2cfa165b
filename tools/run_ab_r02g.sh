#!/bin/bash
# Register kernel for 9 <= n <= 16 vs the stash kernel (device time, graph replay).
cd /root/repo; O=gpurun_out/ab_r02g.txt; : > $O
for i in 1 2; do for v in smallnarrow smallwide; do
  for a in "--n 9 --batch 100000" "--n 9 --batch 1000000" "--n 10 --batch 1000000" "--n 12 --batch 100000" "--n 12 --batch 1000000" \
           "--n 9 --batch 1000000 --dtype f32" "--n 12 --batch 1000000 --dtype f32" "--n 16 --batch 100000 --dtype f32" "--n 16 --batch 1000000 --dtype f32" "--n 14 --batch 1000000 --dtype f32"; do
    python tools/fake_time.py fakebuild/librd_$v.so $a --strategy thread --graph >> $O 2>&1; done
done; done
cat $O
