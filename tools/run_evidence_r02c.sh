#!/bin/bash
# Round-2 evidence refresh at HEAD: GPU suite, smoke, bench lines of every config, the
# launch list of the default bench, ncu --set full of the dominant kernels, sanitizers.
# Output: gpurun_out/ev02c/ (bench lines, logs) and gpurun_out/ncu/ (summaries).
cd /root/repo
R=gpurun_out/ev02c; mkdir -p $R gpurun_out/ncu
timeout 1500 python -m pytest tests -m gpu -q > $R/pytest_gpu.txt 2>&1; tail -3 $R/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $R/smoke.txt 2>&1; tail -1 $R/smoke.txt
timeout 600 python bench.py > $R/bench_C3_f64.json 2> $R/bench_C3_f64.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > $R/bench_reference.json 2>&1
timeout 300 python bench.py --dtype f32 --no-cpu-baseline > $R/bench_C3_f32.json 2>&1
timeout 300 python bench.py --config C2 --steps 500 --no-cpu-baseline > $R/bench_C2_f64.json 2>&1
timeout 300 python bench.py --config C2 --dtype f32 --steps 500 --no-cpu-baseline > $R/bench_C2_f32.json 2>&1
timeout 300 python bench.py --config C4 --steps 50 --cpu-seconds 10 > $R/bench_C4_fd.json 2>&1
timeout 300 python bench.py --config C4 --dtype f32 --steps 50 --no-cpu-baseline > $R/bench_C4_fd_f32.json 2>&1
timeout 300 python bench.py --config C5 --steps 20 --no-cpu-baseline --e2e-steps 1 > $R/bench_C5_f64.json 2>&1
timeout 300 python bench.py --config C1 --steps 200 --no-cpu-baseline > $R/bench_C1_f64.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $R/launches_C3.csv \
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
bash tools/run_ncu_one.sh thread_C3_f64 rnea_thread --config C3 --strategy thread --reps 3 > /dev/null 2>&1
bash tools/run_ncu_one.sh small_C3_f32 rnea_small --config C3 --strategy thread --dtype f32 --reps 3 > /dev/null 2>&1
bash tools/run_ncu_one.sh small_C2_f64 rnea_small --config C2 --reps 3 > /dev/null 2>&1
bash tools/run_ncu_one.sh small_C2_f32 rnea_small --config C2 --dtype f32 --reps 3 > /dev/null 2>&1
bash tools/run_ncu_one.sh aba_C4_f64 aba_dh --config C4 --fd --reps 2 > /dev/null 2>&1
bash tools/run_ncu_one.sh aba_C4_f32 aba_dh --config C4 --fd --dtype f32 --reps 2 > /dev/null 2>&1
bash tools/run_ncu_one.sh rev_n100_1e6_f64 rnea_rev --config C4 --strategy reverse --batch 1000000 --reps 2 > /dev/null 2>&1
for f in $R/bench_*.json; do echo "$f $(python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d.get('value'), d.get('ms_per_step'), (d.get('roofline') or {}).get('frac'))" 2>&1)"; done
for f in gpurun_out/ncu/*.ncu-rep; do [ "$(basename $f)" = "thread_C3_f64.ncu-rep" ] || rm -f $f; done
for tool in memcheck racecheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > $R/sanitizer_$tool.txt 2>&1
  echo "exit $?" >> $R/sanitizer_$tool.txt; tail -3 $R/sanitizer_$tool.txt
done
SKIP_STASH=1 timeout 1500 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_run.py > $R/sanitizer_synccheck_nostash.txt 2>&1
echo "exit $?" >> $R/sanitizer_synccheck_nostash.txt; tail -3 $R/sanitizer_synccheck_nostash.txt
du -sh gpurun_out
