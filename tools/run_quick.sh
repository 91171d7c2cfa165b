#!/bin/bash
# GPU: parity suite + a short ID/FD sweep (args passed to sweep.py)
cd /root/repo; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/gpu_tests.txt
timeout 900 python tools/sweep.py "$@" > gpurun_out/quick_sweep.csv 2>&1
cat gpurun_out/gpu_tests.txt gpurun_out/quick_sweep.csv
