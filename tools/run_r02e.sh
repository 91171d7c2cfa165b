#!/bin/bash
# GPU suite on the product build + the short-chain AUTO grid (device time, graph replay).
cd /root/repo; mkdir -p gpurun_out; O=gpurun_out/r02e.txt; : > $O
echo "== tests: $(timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4)" >> $O
for dt in f64 f32; do
  timeout 1200 python tools/grid_time.py --n 2,3,4,5,6,7,8 --B 256,1024,2048,4096,8192,16384,32768,65536,131072,262144,1000000 \
    --strategies thread,warp_scan,reverse --dtype $dt > gpurun_out/small_grid_$dt.csv 2>&1
done
cat $O
