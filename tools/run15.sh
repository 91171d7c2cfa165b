timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu 2>&1 | grep -E "FAILED|Error|assert|passed|failed" | head -20
