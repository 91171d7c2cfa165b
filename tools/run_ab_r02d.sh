#!/bin/bash
# ABA: TMEM stash of the tip-most records vs ring-only; FD parity on the TMEM build; ncu DRAM.
cd /root/repo; mkdir -p gpurun_out/ncu; O=gpurun_out/ab_r02d.txt; : > $O
for i in 1 2 3; do for v in small3 abatm; do
  for a in "--config C4 --fd" "--config C4 --fd --dtype f32" "--n 30 --batch 100000 --fd" "--n 200 --batch 20000 --fd" "--n 10 --batch 1000000 --fd"; do
    python tools/fake_time.py fakebuild/librd_$v.so $a --graph >> $O 2>&1; done
done; done
cat $O
for v in small3 nosmall; do echo "== diag $v"; python tools/diag_small.py fakebuild/librd_$v.so; done >> $O 2>&1
cp fakebuild/librd_abatm.so paper_1609_04493_b200/librd.so
echo "== fd tests: $(timeout 1500 python -m pytest tests -m gpu -x -q -k 'fd or aba or forward or status or bnd or boundary' 2>&1 | tail -3)" >> $O
bash tools/run_ncu_one.sh aba_C4_f64_tmem aba_dh --config C4 --fd --reps 2 > /dev/null 2>&1
head -30 gpurun_out/ncu/aba_C4_f64_tmem.summary.txt >> $O
tail -40 $O
