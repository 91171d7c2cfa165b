#!/bin/bash
# WS kernel first check: parity + C3 device time vs the current build.
cd /root/repo; R=gpurun_out/ws1; mkdir -p $R
timeout 300 python tools/ws_check.py fakebuild/librd_ws.so > $R/ws.txt 2>&1; tail -20 $R/ws.txt
timeout 120 python tools/ws_check.py paper_1609_04493_b200/librd.so --n 30 --batch 1000 > $R/base.txt 2>&1; tail -2 $R/base.txt
