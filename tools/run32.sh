RD_PP_UNROLL=2 timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "C3 or ragged or link_counts or boundary or many or C2" 2>&1 | tail -1
for i in 1 2; do for v in 1 2; do echo "UNR=$v"; RD_PP_UNROLL=$v timeout 300 python tools/quick_time.py 2>&1 | grep -E "C3 float(64|32) thread|C2 float64 thread"; done; done
