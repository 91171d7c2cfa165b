timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu 2>&1 | grep -E "FAILED|Error|assert|passed|failed" | head
timeout 900 python tools/sweep.py --id-n 10,30 --batches 1000,10000,100000,1000000 --fd-n 10 --fd-batches 1000 --cpu-seconds 0.2 2>&1 | grep "^ID" 
