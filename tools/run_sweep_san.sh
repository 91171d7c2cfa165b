#!/bin/bash
cd /root/repo; mkdir -p gpurun_out/evidence gpurun_out/san
timeout 3000 python tools/sweep.py > gpurun_out/evidence/sweep_f64.csv 2> gpurun_out/evidence/sweep_f64.err
bash tools/run_sanitize.sh
tail -3 gpurun_out/evidence/sweep_f64.err
