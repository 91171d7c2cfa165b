timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu 2>&1 | grep -E "FAILED|Error|passed|failed" | head
timeout 600 python tools/latency.py 2>&1 | head -20
