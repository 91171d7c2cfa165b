mkdir -p gpurun_out/r01
python bench.py > gpurun_out/r01/bench_default.json 2> gpurun_out/r01/bench_default.err
cat gpurun_out/r01/bench_default.json
python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/r01/bench_reference.json 2>&1
cat gpurun_out/r01/bench_reference.json
python bench.py --dtype f32 --no-cpu-baseline > gpurun_out/r01/bench_f32.json 2>&1
python bench.py --config C4 --no-cpu-baseline --steps 50 > gpurun_out/r01/bench_c4.json 2>&1
python bench.py --config C2 --no-cpu-baseline --steps 200 > gpurun_out/r01/bench_c2.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/r01/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r01/bench_under_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:rnea_thread -s 2 -c 1 -o gpurun_out/r01/rnea_thread_pp_c3_f64 python tools/prof_one.py --strategy thread --reps 3 > gpurun_out/r01/ncu_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:aba -s 1 -c 1 -o gpurun_out/r01/aba_c4_f64 python tools/prof_one.py --config C4 --fd --reps 2 > gpurun_out/r01/ncu_aba.log 2>&1
ls -la gpurun_out/r01
