#!/bin/bash
# Device-time grid (CUDA-graph replay) behind the AUTO strategy table, DH chains.
cd /root/repo; mkdir -p gpurun_out/r02
o=gpurun_out/r02/auto_grid_f64.csv
timeout 1200 python tools/grid_time.py --n 7,16,20,30 --B 1,64,256,1000,2048,4096,8192,16384,32768,65536 \
  --strategies thread,warp_scan,reverse,block_scan,chunk:2,chunk:4,chunk:8,chunk:16 > $o 2> $o.err
timeout 1200 python tools/grid_time.py --n 48,64,100,150,200,300,512 --B 1,64,256,1000,2048,4096,8192,16384,32768,65536 \
  --strategies reverse,block_scan,chunk:2,chunk:4,chunk:8,chunk:16,chunk:32 | tail -n +2 >> $o 2>> $o.err
o=gpurun_out/r02/auto_grid_f32.csv
timeout 1200 python tools/grid_time.py --dtype f32 --n 7,30,64,100,200 --B 1,256,1000,4096,16384,65536 \
  --strategies thread,warp_scan,reverse,block_scan,chunk:2,chunk:4,chunk:8,chunk:16,chunk:32 > $o 2> $o.err
