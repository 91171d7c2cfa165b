RD_L1PF=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "C3 or ragged or link_counts or boundary" 2>&1 | tail -1
for i in 1 2; do for v in 0 1; do echo "L1PF=$v"; RD_L1PF=$v timeout 300 python tools/quick_time.py 2>&1 | grep -E "C3 float(64|32) thread|C2 float64 thread"; done; done
