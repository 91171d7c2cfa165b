#!/bin/bash
# thread-kernel knob A/B: C3 / C5-slice / C2 (fp64)
cd /root/repo; mkdir -p gpurun_out
for i in 1 2 3; do for v in $*; do for a in "--config C3" "--config C2" "--n 15 --batch 1000000"; do
  python tools/fake_time.py fakebuild/librd_$v.so $a; done; done; done > gpurun_out/ab6.txt 2>&1
cat gpurun_out/ab6.txt
