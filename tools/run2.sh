mkdir -p gpurun_out/ncu
ncu --set full --clock-control none --import-source on -k regex:rnea_generic -s 1 -c 1 -o gpurun_out/ncu/gen_c3_f64 python tools/prof_one.py --strategy generic --reps 2 > gpurun_out/ncu/gen.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:rnea_thread_tmem -s 1 -c 1 -o gpurun_out/ncu/tmem_c3_f64 python tools/prof_one.py --strategy thread --reps 2 > gpurun_out/ncu/tmem.log 2>&1
RD_STASH=local ncu --set full --clock-control none --import-source on -k regex:rnea_thread_local -s 1 -c 1 -o gpurun_out/ncu/local_c3_f64 python tools/prof_one.py --strategy thread --reps 2 > gpurun_out/ncu/local.log 2>&1
ls -la gpurun_out/ncu
