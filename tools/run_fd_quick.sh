#!/bin/bash
# GPU: parity suite + FD timing of every algorithm at n = 10 / 30, B = 1e3 / 1e5.
cd /root/repo; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/gpu_tests.txt
timeout 600 python tools/sweep.py --id-n 30 --batches 1000 --fd-n 10,30 --fd-batches 1000,100000 --cpu-seconds 0.5 > gpurun_out/fd_sweep.csv 2>&1
cat gpurun_out/gpu_tests.txt gpurun_out/fd_sweep.csv
