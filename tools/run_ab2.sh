#!/bin/bash
# A/B of two variant libraries over the ID configs + the crossover sweep and GPU
# suite on the second one.  usage: tools/run_ab2.sh OLD NEW   (fakebuild/librd_<v>.so)
cd /root/repo; mkdir -p gpurun_out
o=$1; nw=$2
for i in 1 2; do for v in $o $nw; do for a in "--config C3" "--config C5" "--config C2" "--config C2 --dtype f32" "--config C3 --dtype f32" "--config C3 --batch 100000" "--config C3 --batch 20000" "--config C2 --batch 10000"; do
  python tools/fake_time.py fakebuild/librd_$v.so $a; done; done; done > gpurun_out/ab2.txt 2>&1
cp fakebuild/librd_$nw.so paper_1609_04493_b200/librd.so
echo "== tests $nw: $(timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1)" >> gpurun_out/ab2.txt
timeout 600 python tools/crossover.py > gpurun_out/crossover_$nw.csv 2>&1
cat gpurun_out/ab2.txt
