#!/bin/bash
# n = 7 fp64 register kernel: 4 (product) vs 5 / 6 resident CTAs per SM (C2 = 1e5 states in one wave at 6).
cd /root/repo; O=gpurun_out/ab_cap7.txt; : > $O
for rep in 1 2; do for v in base cap5 cap6; do
  cp fakebuild/librd_$v.so paper_1609_04493_b200/librd.so
  python bench.py --config C2 --steps 500 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v bench C2 f64 ms/step', round(d['ms_per_step']*1e3,2), 'us')" >> $O
  python tools/fake_time.py fakebuild/librd_$v.so --config C2 --graph >> $O 2>&1
  python tools/fake_time.py fakebuild/librd_$v.so --n 7 --batch 1000000 --graph >> $O 2>&1
  python tools/fake_time.py fakebuild/librd_$v.so --n 7 --batch 20000 --graph >> $O 2>&1
done; done
cp fakebuild/librd_base.so paper_1609_04493_b200/librd.so
cat $O
