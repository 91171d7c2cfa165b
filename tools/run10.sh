timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | grep -E "FAILED|Error|assert|passed|failed" | head -20
python -c "import __graft_entry__ as g; g.smoke()"
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 1 --steps 50 --warmup 3 --no-cpu-baseline --gather 2>&1 | tail -1 | cut -c1-400
python bench.py --steps 200 --warmup 10 2>&1 | tail -1
