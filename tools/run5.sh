timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -3
RD_PIPE=0 timeout 300 python tools/quick_time.py 2>&1 | grep thread
RD_PIPE=1 timeout 300 python tools/quick_time.py 2>&1 | grep thread
