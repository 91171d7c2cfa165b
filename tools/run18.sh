mkdir -p gpurun_out/ncu
ncu --set full --clock-control none --import-source on -k regex:aba -s 1 -c 1 -o gpurun_out/ncu/aba_v2 python tools/prof_one.py --config C4 --fd --reps 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:rnea_rev -s 1 -c 1 -o gpurun_out/ncu/rev_n100 python tools/prof_one.py --config C4 --reps 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:rnea_thread -s 2 -c 1 -o gpurun_out/ncu/thread_dh python tools/prof_one.py --strategy thread --reps 3 > /dev/null 2>&1
ls gpurun_out/ncu
