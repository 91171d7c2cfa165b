#!/bin/bash
# Register ID kernel: L2 prefetch of the next wave's inputs vs none.
cd /root/repo; O=gpurun_out/ab_pf.txt; : > $O
for rep in 1 2; do for v in base pf; do
  cp fakebuild/librd_$v.so paper_1609_04493_b200/librd.so
  python bench.py --config C2 --steps 500 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v bench C2 f64 ms/step', round(d['ms_per_step']*1e3,2), 'us')" >> $O
  python bench.py --config C3 --dtype f32 --steps 100 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v bench C3 f32 kernel_ms', round(d['roofline']['kernel_ms'],4), 'frac', round(d['roofline']['frac'],3))" >> $O
  python tools/fake_time.py fakebuild/librd_$v.so --config C2 --graph >> $O 2>&1
  python tools/fake_time.py fakebuild/librd_$v.so --config C2 --dtype f32 --graph >> $O 2>&1
  for n in 7 12; do python tools/fake_time.py fakebuild/librd_$v.so --n $n --batch 1000000 --graph >> $O 2>&1; done
  for n in 16 30; do python tools/fake_time.py fakebuild/librd_$v.so --n $n --batch 1000000 --dtype f32 --graph >> $O 2>&1; done
done; done
cp fakebuild/librd_pf.so paper_1609_04493_b200/librd.so
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "short_chain or C2 or C3" >> $O 2>&1
cp fakebuild/librd_base.so paper_1609_04493_b200/librd.so
cat $O
