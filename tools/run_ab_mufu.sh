#!/bin/bash
# fp32 register ID kernel / REVERSE: sin/cos on the SFU (MUFU) vs the polynomial.
cd /root/repo; O=gpurun_out/ab_mufu.txt; : > $O
for rep in 1 2; do for v in base mufu; do
  for n in 7 12 20 30; do python tools/fake_time.py fakebuild/librd_$v.so --n $n --batch 1000000 --dtype f32 --graph >> $O 2>&1; done
  python tools/fake_time.py fakebuild/librd_$v.so --n 100 --batch 1000000 --dtype f32 --strategy reverse --graph >> $O 2>&1
done; done
cp fakebuild/librd_mufu.so paper_1609_04493_b200/librd.so
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "float32" 2>&1 | tail -3 >> $O
python tools/f32_accuracy.py >> $O 2>&1
cp fakebuild/librd_base.so paper_1609_04493_b200/librd.so
cat $O
