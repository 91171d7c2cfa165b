timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -5
timeout 300 python tools/quick_time.py 2>&1 | tee gpurun_out/qt_v4.txt
