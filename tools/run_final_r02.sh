#!/bin/bash
# Round-2 final check at HEAD: GPU suite, smoke, default bench line, reference arm, C4 line.
cd /root/repo; R=gpurun_out/final; mkdir -p $R
timeout 1500 python -m pytest tests -m gpu -q > $R/pytest_gpu.txt 2>&1; tail -2 $R/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $R/smoke.txt 2>&1; tail -1 $R/smoke.txt
timeout 600 python bench.py > $R/bench_C3_f64.json 2> $R/bench_C3_f64.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > $R/bench_reference.json 2>&1
timeout 300 python bench.py --config C4 --steps 50 --cpu-seconds 10 > $R/bench_C4_fd.json 2>&1
for f in $R/bench_*.json; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d.get('value'), d.get('ms_per_step'), (d.get('roofline') or {}).get('frac'), (d.get('e2e') or {}).get('value'))"; done
