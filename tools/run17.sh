timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu 2>&1 | grep -E "FAILED|Error|assert|passed|failed" | head -20
timeout 900 python tools/sweep.py --id-n 30,100,200 --batches 100000,1000000 --fd-n 30,100 --fd-batches 100000 --cpu-seconds 0.5 2>&1 | grep -v "^ID,warp"
