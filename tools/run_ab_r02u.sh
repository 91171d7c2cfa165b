#!/bin/bash
# Register ABA (short chains) vs the workspace ABA kernel; fp64 register caps; then the GPU suite.
cd /root/repo; O=gpurun_out/ab_r02u.csv; echo "lib,dtype,n,B,ms" > $O
for v in noabas abas abas3 abas4; do for dt in f64 f32; do for n in 2 4 6 7 8 10 12; do for B in 100000 1000000; do
  [ $dt = f32 ] && [ $v != noabas ] && [ $v != abas ] && continue
  python tools/fake_time.py fakebuild/librd_$v.so --n $n --batch $B --dtype $dt --fd --graph 2>&1 | awk -v v=$v -v d=$dt -v n=$n -v B=$B '/ ms$/{print v","d","n","B","$(NF-1)}' >> $O
done; done; done; done
cat $O
echo "== tests: $(timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4)"
