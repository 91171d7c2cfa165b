#!/bin/bash
# After tools/run_ab_fd.sh: C4 bench line + ncu capture of the ABA kernel with the in-tree librd.so.
cd /root/repo; R=gpurun_out/evidence2; mkdir -p $R gpurun_out/ncu
python bench.py --config C4 --steps 50 --cpu-seconds 10 > $R/bench_C4_fd.json 2>&1
bash tools/run_ncu_one.sh aba_C4_f64 aba_dh --config C4 --fd --reps 2 > /dev/null 2>&1
cat $R/bench_C4_fd.json; head -20 gpurun_out/ncu/aba_C4_f64.summary.txt
