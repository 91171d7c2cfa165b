#!/bin/bash
# WS kernel: parity + C3 device time, then one ncu capture.
cd /root/repo; R=gpurun_out/ws3; mkdir -p $R
timeout 300 python tools/ws_check.py fakebuild/librd_ws.so --n 4,6,16,20,22,30,32 > $R/ws.txt 2>&1; tail -4 $R/ws.txt
bash tools/run_ncu_one.sh ws_C3 rnea_ws --config C3 --strategy thread --reps 2 --lib fakebuild/librd_ws.so > /dev/null 2>&1
head -30 gpurun_out/ncu/ws_C3.summary.txt
