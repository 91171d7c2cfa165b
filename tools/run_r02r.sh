#!/bin/bash
# fp64 n = 13..16 small batches: register kernel vs the scans (AUTO), then cold-C2 caps.
cd /root/repo
timeout 900 python tools/grid_time.py --n 13,14,16 --B 256,1024,1536,2048,4096,16384,65536,262144 \
  --strategies thread,warp_scan,chunk:8,chunk:4,reverse --dtype f64 > gpurun_out/small_grid4_f64.csv 2>&1
bash tools/run_ab_r02q.sh
