#!/bin/bash
# A/B over several argument sets: tools/run_ab_multi.sh "v1 v2" "args1" "args2" ...  (then GPU tests per variant)
cd /root/repo; mkdir -p gpurun_out
vs=$1; shift
: > gpurun_out/ab.txt
for i in 1 2; do for a in "$@"; do for v in $vs; do python tools/fake_time.py fakebuild/librd_$v.so $a >> gpurun_out/ab.txt 2>&1; done; done; done
cp paper_1609_04493_b200/librd.so /tmp/librd_orig.so
for v in $vs; do
  cp fakebuild/librd_$v.so paper_1609_04493_b200/librd.so
  echo "== tests $v: $(timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1)" >> gpurun_out/ab.txt
done
cp /tmp/librd_orig.so paper_1609_04493_b200/librd.so
sort gpurun_out/ab.txt | uniq -c | sort -k2 | head -0
cat gpurun_out/ab.txt
