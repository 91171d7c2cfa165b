set -x
nvidia-smi --query-gpu=name,clocks.sm --format=csv
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -30 > gpurun_out/pytest_gpu.txt
cat gpurun_out/pytest_gpu.txt
RD_STASH=tmem timeout 300 python tools/quick_time.py 2>&1 | tee gpurun_out/qt_tmem.txt
RD_STASH=local timeout 300 python tools/quick_time.py 2>&1 | tee gpurun_out/qt_local.txt
