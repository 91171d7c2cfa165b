#!/bin/bash
# Evidence pass: bench lines, reference arm, ncu launch list + full captures, sweeps.
# Output: gpurun_out/evidence/ (copy what is judged into profiles/rNN/).
cd /root/repo
R=gpurun_out/evidence
mkdir -p $R gpurun_out/ncu
python bench.py > $R/bench_C3_f64.json 2> $R/bench_C3_f64.err
python bench.py --impl reference --steps 20 --warmup 3 > $R/bench_reference.json 2>&1
python bench.py --dtype f32 --no-cpu-baseline > $R/bench_C3_f32.json 2>&1
python bench.py --config C4 --steps 50 --cpu-seconds 10 > $R/bench_C4_fd.json 2>&1
python bench.py --config C2 --steps 500 --no-cpu-baseline > $R/bench_C2_f64.json 2>&1
python bench.py --config C2 --dtype f32 --steps 500 --no-cpu-baseline > $R/bench_C2_f32.json 2>&1
python bench.py --config C5 --steps 20 --no-cpu-baseline --e2e-steps 1 > $R/bench_C5_f64.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $R/launches_C3.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
bash tools/run_ncu_one.sh thread_C3_f64 rnea_thread --config C3 --strategy thread --reps 3 > /dev/null 2>&1
bash tools/run_ncu_one.sh thread_C3_f32 rnea_thread --config C3 --strategy thread --dtype f32 --reps 3 > /dev/null 2>&1
bash tools/run_ncu_one.sh aba_C4_f64 aba_dh --config C4 --fd --reps 2 > /dev/null 2>&1
bash tools/run_ncu_one.sh rev_n100_f64 rnea_rev --config C4 --strategy reverse --reps 2 > /dev/null 2>&1
bash tools/run_ncu_one.sh warp_C3_f64 rnea_warp_kernel --strategy warp_scan --batch 100000 --reps 2 > /dev/null 2>&1
timeout 2400 python tools/sweep.py > $R/sweep_f64.csv 2> $R/sweep_f64.err
timeout 900 python tools/sweep.py --dtype f32 --fd-n 10,30 --cpu-seconds 1 > $R/sweep_f32.csv 2> $R/sweep_f32.err
timeout 600 python tools/latency.py > $R/latency.csv 2>&1
timeout 300 python tools/small_probe.py C2 C3 > $R/small_probe.csv 2>&1
ls -la $R gpurun_out/ncu
