#!/bin/bash
# Re-entry check of HEAD: GPU suite, smoke, default bench line.
cd /root/repo; R=gpurun_out/head2; mkdir -p $R
timeout 1500 python -m pytest tests -m gpu -q -x > $R/pytest_gpu.txt 2>&1; tail -3 $R/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $R/smoke.txt 2>&1; tail -1 $R/smoke.txt
timeout 600 python bench.py > $R/bench_C3_f64.json 2> $R/bench_C3_f64.err; cat $R/bench_C3_f64.json
