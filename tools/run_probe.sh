cd /root/repo; mkdir -p gpurun_out
timeout 300 python tools/small_probe.py C2 C3 > gpurun_out/small_probe.csv 2>&1
bash tools/run_ncu_one.sh c2_thread_f64 rnea_thread --config C2 --strategy thread > /dev/null 2>&1
bash tools/run_ncu_one.sh c2_thread_f32 rnea_thread --config C2 --strategy thread --dtype f32 > /dev/null 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 20 --warmup 3 > gpurun_out/torchrun1.json 2> gpurun_out/torchrun1.err
cat gpurun_out/small_probe.csv; cat gpurun_out/ncu/c2_thread_f64.summary.txt | head -40; cat gpurun_out/torchrun1.json; tail -3 gpurun_out/torchrun1.err
