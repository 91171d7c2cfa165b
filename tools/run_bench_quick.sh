#!/bin/bash
cd /root/repo; R=gpurun_out/bq; mkdir -p $R
python bench.py --no-cpu-baseline --e2e-steps 1 > $R/C3.json 2>&1
python bench.py --dtype f32 --no-cpu-baseline --e2e-steps 0 > $R/C3f32.json 2>&1
python bench.py --config C5 --steps 20 --no-cpu-baseline --e2e-steps 0 > $R/C5.json 2>&1
python bench.py --config C2 --steps 500 --no-cpu-baseline --e2e-steps 0 > $R/C2.json 2>&1
for f in $R/*.json; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['value'], d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['clocks'])"; done
