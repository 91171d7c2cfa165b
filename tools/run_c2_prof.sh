#!/bin/bash
# C2 (n = 7, 1e5 states) ncu captures, fp64 and fp32, and the launch list of the bench.
cd /root/repo; mkdir -p gpurun_out/ncu
bash tools/run_ncu_one.sh thread_C2_f64 rnea_thread --config C2 --reps 3 > /dev/null 2>&1
bash tools/run_ncu_one.sh thread_C2_f32 rnea_thread --config C2 --dtype f32 --reps 3 > /dev/null 2>&1
head -40 gpurun_out/ncu/thread_C2_f64.summary.txt
head -20 gpurun_out/ncu/thread_C2_f32.summary.txt
