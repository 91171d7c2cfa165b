#!/bin/bash
# ncu --set full summaries of the secondary strategies, each in the regime AUTO picks it
# (north_star (4): every strategy choice evidenced by pipe / occupancy / DRAM counters).
cd /root/repo; mkdir -p gpurun_out/ncu
bash tools/run_ncu_one.sh warp_scan_n30_B4096 rnea_warp --config C3 --strategy warp_scan --batch 4096 --reps 3 > /dev/null 2>&1
bash tools/run_ncu_one.sh block_scan_n256_B1 rnea_block --n 256 --strategy block_scan --batch 1 --reps 3 > /dev/null 2>&1
bash tools/run_ncu_one.sh chunk8_n100_B1000 rnea_chunk --n 100 --strategy chunk:8 --batch 1000 --reps 3 > /dev/null 2>&1
bash tools/run_ncu_one.sh small_n12_1e6_f64 rnea_small --n 12 --strategy thread --batch 1000000 --reps 2 > /dev/null 2>&1
bash tools/run_ncu_one.sh aba_small_n7_1e6_f64 aba_small --n 7 --fd --batch 1000000 --reps 2 > /dev/null 2>&1
bash tools/run_ncu_one.sh jsiia_n30_B10000 jsiia --n 30 --fd --fd-algo jsiia --batch 10000 --reps 2 > /dev/null 2>&1
bash tools/run_ncu_one.sh rev_n100_1e6_f32 rnea_rev --config C4 --strategy reverse --batch 1000000 --dtype f32 --reps 2 > /dev/null 2>&1
rm -f gpurun_out/ncu/*.ncu-rep
for f in gpurun_out/ncu/*.summary.txt; do echo "== $f"; sed -n 1,13p $f; done
