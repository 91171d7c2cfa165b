#!/bin/bash
cd /root/repo
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "joint_frames or screw or nearly_parallel or auto_strategy or host_path" 2>&1 | tail -3
python tools/jf_time.py 2>&1 | tee gpurun_out/jf_time2.csv
