timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu 2>&1 | tail -1
RD_RING=0 timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "C3 or ragged or many" 2>&1 | tail -1
for i in 1 2; do for v in 0 1; do echo "RING=$v"; RD_RING=$v timeout 300 python tools/quick_time.py 2>&1 | grep -E "C3 float(64|32) thread|C2 float64 thread"; done; done
