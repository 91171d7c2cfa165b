#!/bin/bash
cd /root/repo
for v in base jf; do cp fakebuild/librd_$v.so paper_1609_04493_b200/librd.so; echo "== $v"; python tools/jf_fd_time.py 2>&1; done | tee gpurun_out/jf_fd_ab.txt
cp fakebuild/librd_jf.so paper_1609_04493_b200/librd.so
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fd or nearly_parallel or screw" 2>&1 | tail -3
