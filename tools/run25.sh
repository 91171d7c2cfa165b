mkdir -p gpurun_out/r01
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu 2>&1 | grep -E "FAILED|Error|assert|passed|failed" | head
timeout 600 python tools/latency.py > gpurun_out/r01/latency.csv 2>&1
