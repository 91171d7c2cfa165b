#!/bin/bash
# Short-chain register kernel A/B (device time, graph replay) + GPU suite on the product build.
cd /root/repo; mkdir -p gpurun_out; O=gpurun_out/ab_r02c.txt; : > $O
for i in 1 2; do for v in nosmall small2 small3 small4; do
  L=fakebuild/librd_$v.so
  for a in "--config C2" "--config C2 --dtype f32" "--config C2 --batch 1000000" "--n 8 --batch 100000" "--n 4 --batch 100000" "--n 8 --batch 1000000 --dtype f32"; do
    python tools/fake_time.py $L $a --strategy thread --graph >> $O 2>&1; done
done; done
cat $O
echo "== tests: $(timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3)" >> $O
tail -4 $O
