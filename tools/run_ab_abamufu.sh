#!/bin/bash
# fp32 ABA (workspace kernel and register ABA): SFU sin/cos vs polynomial.
cd /root/repo; O=gpurun_out/ab_abamufu.txt; : > $O
for rep in 1 2; do for v in base abamufu; do
  python tools/fake_time.py fakebuild/librd_$v.so --config C4 --fd --dtype f32 --graph >> $O 2>&1
  for n in 7 16 30; do python tools/fake_time.py fakebuild/librd_$v.so --n $n --batch 1000000 --fd --dtype f32 --graph >> $O 2>&1; done
done; done
cp fakebuild/librd_abamufu.so paper_1609_04493_b200/librd.so
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "fd" 2>&1 | tail -2 >> $O
python tools/long_chain_fd_accuracy.py >> $O 2>&1
cp fakebuild/librd_base.so paper_1609_04493_b200/librd.so
cat $O
