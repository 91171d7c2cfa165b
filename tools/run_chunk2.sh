#!/bin/bash
cd /root/repo; mkdir -p gpurun_out/r02
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -k "chunk" 2>&1 | tail -5 > gpurun_out/r02/chunk_parity2.txt
timeout 900 python tools/grid_time.py --n 30,100,200 --B 1000,4096,16384,65536,1000000 \
  --strategies reverse,chunk:2,chunk:4,chunk:8,chunk:16,chunk:32 > gpurun_out/r02/chunk_grid2_f64.csv 2> gpurun_out/r02/chunk_grid2.err
timeout 300 python tools/grid_time.py --n 7 --robot arm7 --B 100000 --strategies thread,reverse,chunk:2,warp_scan >> gpurun_out/r02/chunk_grid2_f64.csv 2>> gpurun_out/r02/chunk_grid2.err
