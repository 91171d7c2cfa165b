#!/bin/bash
# GPU suite + the paper-shaped strategy sweep (evals/s vs B, CPU oracle beside) at the final kernels.
cd /root/repo; mkdir -p gpurun_out/sw
echo "== tests: $(timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3)" > gpurun_out/sw/tests.txt
cat gpurun_out/sw/tests.txt
timeout 2400 python tools/sweep.py > gpurun_out/sw/sweep_f64.csv 2> gpurun_out/sw/sweep_f64.err
timeout 1200 python tools/sweep.py --dtype f32 --fd-n 10,30 --cpu-seconds 1 > gpurun_out/sw/sweep_f32.csv 2> gpurun_out/sw/sweep_f32.err
wc -l gpurun_out/sw/*.csv
