#!/bin/bash
# A/B timing of variant libraries: tools/run_ab.sh "v1 v2 ..." [fake_time args] (fakebuild/librd_<v>.so),
# then the GPU suite against each variant.  Output in gpurun_out/ab.txt.
cd /root/repo; mkdir -p gpurun_out
vs=$1; shift
for i in 1 2 3; do for v in $vs; do python tools/fake_time.py fakebuild/librd_$v.so "$@"; done; done > gpurun_out/ab.txt 2>&1
cp paper_1609_04493_b200/librd.so /tmp/librd_orig.so
for v in $vs; do
  cp fakebuild/librd_$v.so paper_1609_04493_b200/librd.so
  echo "== tests $v: $(timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1)" >> gpurun_out/ab.txt
done
cp /tmp/librd_orig.so paper_1609_04493_b200/librd.so
cat gpurun_out/ab.txt
