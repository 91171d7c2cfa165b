#!/bin/bash
# REVERSE A/B (OLD NEW) + GPU suite and crossover sweep on NEW.
cd /root/repo; mkdir -p gpurun_out
o=$1; nw=$2
for i in 1 2 3; do for v in $o $nw; do for a in "--n 30 --batch 16384 --strategy reverse" "--n 100 --batch 100000 --strategy reverse" "--n 200 --batch 10000 --strategy reverse" "--n 30 --batch 1000000 --strategy reverse"; do
  python tools/fake_time.py fakebuild/librd_$v.so $a; done; done; done > gpurun_out/ab5.txt 2>&1
cp fakebuild/librd_$nw.so paper_1609_04493_b200/librd.so
echo "== tests $nw: $(timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3)" >> gpurun_out/ab5.txt
timeout 900 python tools/crossover.py > gpurun_out/crossover_$nw.csv 2>&1
cat gpurun_out/ab5.txt
