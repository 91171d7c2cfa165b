#!/bin/bash
# C2 fp64 with a cold L2 (bench.py's own timing) for the register kernel's register caps.
cd /root/repo; O=gpurun_out/ab_r02q.txt; : > $O
cp paper_1609_04493_b200/librd.so /tmp/librd_keep.so
for i in 1 2; do for v in prod cap3 cap4; do
  cp fakebuild/librd_$v.so paper_1609_04493_b200/librd.so
  python bench.py --config C2 --steps 500 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', 'bench C2 f64 ms/step', round(d['ms_per_step']*1e3,2), 'us', 'kernel', round(d['roofline']['kernel_ms']*1e3,2), 'us')" >> $O
  python tools/fake_time.py fakebuild/librd_$v.so --config C2 --graph >> $O 2>&1
  python tools/fake_time.py fakebuild/librd_$v.so --n 7 --batch 1000000 --graph >> $O 2>&1
done; done
cp /tmp/librd_keep.so paper_1609_04493_b200/librd.so
cat $O
