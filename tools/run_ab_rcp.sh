#!/bin/bash
# A/B: ABA pivot reciprocal without the IEEE slow path (rcp_pivot) vs 1 / D.
cd /root/repo; O=gpurun_out/ab_rcp.txt; : > $O
for v in base rcp; do
  for dt in f64 f32; do
    python tools/fake_time.py fakebuild/librd_$v.so --config C4 --fd --dtype $dt --graph >> $O 2>&1
    python tools/fake_time.py fakebuild/librd_$v.so --n 7 --batch 1000000 --fd --dtype $dt --graph >> $O 2>&1
    python tools/fake_time.py fakebuild/librd_$v.so --n 30 --batch 1000000 --fd --dtype $dt --graph >> $O 2>&1
  done
done
cat $O
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/ab_rcp_pytest.txt 2>&1; tail -3 gpurun_out/ab_rcp_pytest.txt
