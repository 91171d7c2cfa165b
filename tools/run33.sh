timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k fd 2>&1 | tail -1
timeout 900 python tools/sweep.py --id-n 10 --batches 1000 --fd-n 30,100,200 --fd-batches 100000 --cpu-seconds 0.2 2>&1 | grep "FD,aba,"
