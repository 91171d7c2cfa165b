timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu 2>&1 | tail -1
for i in 1 2; do timeout 300 python tools/quick_time.py 2>&1 | grep -E "C3 float(64|32) thread"; done
python bench.py 2>&1 | tail -1
