#!/bin/bash
cd /root/repo
python tools/long_chain_accuracy.py 2>&1 | tee gpurun_out/long_chain_accuracy.csv
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
