#!/bin/bash
# Final-config check: GPU suite, C2 bench (cold L2), register-kernel timings.
cd /root/repo; O=gpurun_out/r02t.txt; : > $O
echo "== tests: $(timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3)" >> $O
python bench.py --config C2 --steps 500 --no-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 >> $O
L=paper_1609_04493_b200/librd.so
for a in "--config C2" "--n 7 --batch 1000000" "--n 9 --batch 1000000" "--n 6 --batch 1000000" "--n 14 --batch 100000"; do
  python tools/fake_time.py $L $a --strategy thread --graph >> $O 2>&1; done
cat $O
