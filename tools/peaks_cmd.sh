nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/peaks_clocks.csv &
SMI=$!
./tools/peaks_alu > gpurun_out/peaks_alu.jsonl 2>&1
kill $SMI
nvidia-smi > gpurun_out/nvsmi.txt; lscpu > gpurun_out/lscpu.txt; nproc >> gpurun_out/lscpu.txt
