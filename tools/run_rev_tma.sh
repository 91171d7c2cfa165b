#!/bin/bash
cd /root/repo; mkdir -p gpurun_out/r02
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -k "reverse or ragged or link_counts or prismatic or boundary or wide or large_joint" 2>&1 | tail -5 > gpurun_out/r02/rev_tma_parity.txt
timeout 900 python tools/grid_time.py --n 30,100,200 --B 1000,16384,65536,100000,1000000 --strategies reverse > gpurun_out/r02/rev_tma_grid.csv 2> gpurun_out/r02/rev_tma_grid.err
timeout 300 python tools/grid_time.py --n 100 --B 1000000 --strategies reverse --dtype f32 >> gpurun_out/r02/rev_tma_grid.csv 2>> gpurun_out/r02/rev_tma_grid.err
