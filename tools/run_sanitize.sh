#!/bin/bash
cd /root/repo; mkdir -p gpurun_out/san
for tool in memcheck racecheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > gpurun_out/san/sanitizer_$tool.txt 2>&1
  tail -3 gpurun_out/san/sanitizer_$tool.txt
done
SKIP_STRATS=thread timeout 1500 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_run.py > gpurun_out/san/sanitizer_synccheck_nothread.txt 2>&1
tail -3 gpurun_out/san/sanitizer_synccheck_nothread.txt
