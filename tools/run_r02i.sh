#!/bin/bash
# fp32 register kernel (n <= 32) vs the scan strategies at small batches (AUTO table).
cd /root/repo
timeout 1500 python tools/grid_time.py --n 16,20,24,28,30,32 --B 256,512,1024,2048,4096,8192,16384,32768,65536 \
  --strategies thread,warp_scan,chunk:4,chunk:8,reverse --dtype f32 > gpurun_out/small_grid3_f32.csv 2>&1
timeout 600 python tools/grid_time.py --n 12 --B 1536,2048,3072 --strategies thread,warp_scan,reverse --dtype f64 > gpurun_out/small_grid3_f64.csv 2>&1
tail -3 gpurun_out/small_grid3_f32.csv
