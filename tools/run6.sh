timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -3
RD_PP=0 timeout 300 python tools/quick_time.py 2>&1 | grep thread
RD_PP=1 timeout 300 python tools/quick_time.py 2>&1 | grep thread
RD_PP=0 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "C3 or large" 2>&1 | tail -2
