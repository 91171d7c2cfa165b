#!/bin/bash
cd /root/repo; mkdir -p gpurun_out
python tools/pcie_peak.py > gpurun_out/pcie_peak.txt 2>&1; cat gpurun_out/pcie_peak.txt
python tools/e2e_time.py > gpurun_out/e2e_time.txt 2>&1; tail -5 gpurun_out/e2e_time.txt
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_head3.txt 2>&1; tail -2 gpurun_out/pytest_head3.txt
