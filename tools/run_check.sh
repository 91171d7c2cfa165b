#!/bin/bash
# GPU: full parity suite + quick timings of the default build.
cd /root/repo; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/check.txt
L=paper_1609_04493_b200/librd.so
for a in "--config C3" "--config C3 --dtype f32" "--config C2" "--config C5" "--config C4 --fd" "--config C2 --dtype f32"; do
  python tools/fake_time.py $L $a >> gpurun_out/check.txt 2>&1
done
cat gpurun_out/check.txt
