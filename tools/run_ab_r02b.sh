#!/bin/bash
# C2 device-time A/B (graph replay) of thread-kernel plans + ABA ncu at the new ring config.
cd /root/repo; mkdir -p gpurun_out/ncu; O=gpurun_out/ab_r02b.txt; : > $O
for i in 1 2; do for v in new nte w8; do
  L=fakebuild/librd_$v.so
  for a in "--config C2" "--config C2 --dtype f32" "--config C2 --batch 65536" "--config C3" "--config C3 --batch 200000"; do
    python tools/fake_time.py $L $a --strategy thread --graph >> $O 2>&1; done
  for a in "--config C2" "--config C2 --dtype f32"; do
    python tools/fake_time.py $L $a --strategy reverse --graph >> $O 2>&1; done
done; done
for i in 1 2; do
  for a in "--config C4 --fd" "--config C4 --fd --dtype f32" "--n 30 --batch 100000 --fd" "--n 200 --batch 20000 --fd"; do
    python tools/fake_time.py fakebuild/librd_new.so $a --graph >> $O 2>&1; done; done
cat $O
bash tools/run_ncu_one.sh aba_C4_f64_ring rnea_aba_dh --config C4 --fd --reps 2 > /dev/null 2>&1
bash tools/run_ncu_one.sh aba_C4_f64_ring aba_dh --config C4 --fd --reps 2 > /dev/null 2>&1
head -40 gpurun_out/ncu/aba_C4_f64_ring.summary.txt
