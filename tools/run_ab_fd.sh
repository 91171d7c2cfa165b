#!/bin/bash
# A/B of variant libraries on the FD configs + GPU suite on the last one.
# usage: tools/run_ab_fd.sh "v1 v2 ..."   (fakebuild/librd_<v>.so)
cd /root/repo; mkdir -p gpurun_out
vs=$1
for i in 1 2 3; do for v in $vs; do for a in "--config C4 --fd" "--n 30 --batch 100000 --fd" "--n 200 --batch 100000 --fd"; do
  python tools/fake_time.py fakebuild/librd_$v.so $a; done; done; done > gpurun_out/ab_fd.txt 2>&1
last=${vs##* }
cp fakebuild/librd_$last.so paper_1609_04493_b200/librd.so
echo "== tests $last: $(timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3)" >> gpurun_out/ab_fd.txt
cat gpurun_out/ab_fd.txt
