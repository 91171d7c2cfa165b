#!/bin/bash
# ncu --set full of the kernels this round works on (summaries -> gpurun_out/ncu)
cd /root/repo; mkdir -p gpurun_out/ncu
bash tools/run_ncu_one.sh rev_n100_1M rnea_rev --config C4 --batch 1000000 --strategy reverse --reps 2 > /dev/null 2>&1
bash tools/run_ncu_one.sh aba_C4 aba_dh --config C4 --fd --reps 2 > /dev/null 2>&1
bash tools/run_ncu_one.sh thread_C2_f64 rnea_thread --config C2 --strategy thread --reps 3 > /dev/null 2>&1
bash tools/run_ncu_one.sh chunk_n100_4k rnea_chunk --config C4 --batch 4096 --strategy chunk:8 --reps 3 > /dev/null 2>&1
ls gpurun_out/ncu
