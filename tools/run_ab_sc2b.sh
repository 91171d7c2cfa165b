#!/bin/bash
# fp32 register kernel: paired sin/cos (sc2) vs scalar, every n, 1e6 and 1e5 states.
cd /root/repo; O=gpurun_out/ab_sc2b.csv; echo "lib,n,B,ms" > $O
for v in base sc2; do for B in 1000000 100000; do for n in $(seq 9 32); do
  python tools/fake_time.py fakebuild/librd_$v.so --n $n --batch $B --dtype f32 --graph 2>&1 | awk -v v=$v -v n=$n -v B=$B '/ ms$/{print v","n","B","$(NF-1)}' >> $O
done; done; done
python - <<'PY'
import csv, collections
d=collections.defaultdict(dict)
for r in csv.DictReader(open('gpurun_out/ab_sc2b.csv')): d[(int(r['n']),int(r['B']))][r['lib']]=float(r['ms'])
for k in sorted(d): print(k, d[k].get('base'), d[k].get('sc2'), '%.3f' % (d[k].get('sc2',0)/d[k].get('base',1)))
PY
