timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
cat gpurun_out/pytest_gpu.txt
timeout 300 python tools/quick_time.py 2>&1 | tee gpurun_out/qt_v3.txt
mkdir -p gpurun_out/ncu
ncu --set full --clock-control none --import-source on -k regex:rnea_thread -s 1 -c 1 -o gpurun_out/ncu/thread_v3_c3_f64 python tools/prof_one.py --strategy thread --reps 2 > gpurun_out/ncu/v3.log 2>&1
