#!/bin/bash
cd /root/repo
bash tools/run_ncu_one.sh ws_C3 rnea_ws --config C3 --strategy thread --reps 2 --lib fakebuild/librd_ws.so > /dev/null 2>&1
cat gpurun_out/ncu/ws_C3.summary.txt | head -80
rm -f gpurun_out/ncu/ws_C3.ncu-rep.bak
