#!/bin/bash
# A/B: ABA cp.async ring depths / occupancy, balanced thread-kernel tiles; then the GPU suite.
cd /root/repo; mkdir -p gpurun_out; O=gpurun_out/ab_r02a.txt; : > $O
for i in 1 2; do for v in head new ring4 ring7 ring4mb4; do
  L=fakebuild/librd_$v.so
  for a in "--config C4 --fd" "--config C4 --fd --dtype f32" "--n 30 --batch 100000 --fd" "--n 200 --batch 20000 --fd"; do
    python tools/fake_time.py $L $a >> $O 2>&1; done
done; done
for i in 1 2; do for v in head new; do
  L=fakebuild/librd_$v.so
  for a in "--config C2" "--config C2 --dtype f32" "--config C3" "--config C3 --dtype f32" "--config C2 --batch 65536" "--config C3 --batch 200000"; do
    python tools/fake_time.py $L $a --strategy thread >> $O 2>&1; done
done; done
echo "== tests: $(timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3)" >> $O
cat $O
