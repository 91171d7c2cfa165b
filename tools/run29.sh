RD_ABA_MB=3 timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k fd 2>&1 | tail -1
for v in 2 3 4; do echo MB=$v; RD_ABA_MB=$v timeout 900 python tools/sweep.py --id-n 10 --batches 1000 --fd-n 30,100 --fd-batches 100000 --cpu-seconds 0.2 2>&1 | grep "FD,aba,"; done
