#!/bin/bash
# Product GPU suite; small-kernel AUTO grid for fp64 n = 9..12 / fp32 n = 9..16; fp32 register kernel up to n = 32.
cd /root/repo; O=gpurun_out/r02h.txt; : > $O
echo "== tests: $(timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4)" >> $O
timeout 900 python tools/grid_time.py --n 9,10,11,12 --B 256,1024,4096,16384,65536,262144,400000 --strategies thread,warp_scan,reverse --dtype f64 > gpurun_out/small_grid2_f64.csv 2>&1
timeout 900 python tools/grid_time.py --n 9,12,16,17 --B 256,1024,4096,16384,65536,262144,1000000 --strategies thread,warp_scan,reverse --dtype f32 > gpurun_out/small_grid2_f32.csv 2>&1
for i in 1 2; do for v in prod f32w32; do
  for a in "--n 20 --batch 1000000" "--n 24 --batch 1000000" "--n 28 --batch 1000000" "--n 30 --batch 1000000" "--n 32 --batch 1000000" "--n 24 --batch 100000" "--n 30 --batch 100000"; do
    python tools/fake_time.py fakebuild/librd_$v.so $a --dtype f32 --strategy thread --graph >> $O 2>&1; done
done; done
cat $O
