#!/bin/bash
# GPU: CHUNK parity + timing grid against THREAD / REVERSE / BLOCK_SCAN.
cd /root/repo; mkdir -p gpurun_out/r02
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -k "chunk or ragged or C3_small" 2>&1 | tail -25 > gpurun_out/r02/chunk_parity.txt
timeout 900 python tools/grid_time.py --n 7,30,100,200 --B 1000,4096,16384,65536,262144,1000000 \
  --strategies thread,reverse,block_scan,chunk:2,chunk:4,chunk:8,chunk:16,chunk:32 > gpurun_out/r02/chunk_grid_f64.csv 2> gpurun_out/r02/chunk_grid.err
