#!/bin/bash
# Round-2 HEAD check: gpu parity suite, smoke, bench lines for C3/C2/C4.
cd /root/repo; R=gpurun_out/r02head; mkdir -p $R
timeout 1500 python -m pytest tests -m gpu -x -q > $R/pytest_gpu.txt 2>&1; tail -3 $R/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $R/smoke.txt 2>&1; tail -1 $R/smoke.txt
timeout 600 python bench.py > $R/bench_C3_f64.json 2> $R/bench_C3_f64.err; cat $R/bench_C3_f64.json
timeout 300 python bench.py --config C2 --steps 500 --no-cpu-baseline > $R/bench_C2_f64.json 2>&1
timeout 300 python bench.py --config C2 --dtype f32 --steps 500 --no-cpu-baseline > $R/bench_C2_f32.json 2>&1
timeout 300 python bench.py --dtype f32 --no-cpu-baseline > $R/bench_C3_f32.json 2>&1
timeout 300 python bench.py --config C4 --steps 50 --no-cpu-baseline > $R/bench_C4_fd.json 2>&1
for f in $R/bench_*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d.get('roofline',{}).get('frac'))"; done
