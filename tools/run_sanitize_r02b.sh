#!/bin/bash
# Sanitizers at the final round-2 build: every kernel incl. the register THREAD kernel and
# the cp.async ABA ring; synccheck on everything but the TMEM stash kernel (tool limitation).
cd /root/repo; R=gpurun_out/san02b; mkdir -p $R
for tool in memcheck racecheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > $R/sanitizer_$tool.txt 2>&1
  echo "exit $?" >> $R/sanitizer_$tool.txt; tail -3 $R/sanitizer_$tool.txt
done
SKIP_STASH=1 timeout 1500 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_run.py > $R/sanitizer_synccheck_nostash.txt 2>&1
echo "exit $?" >> $R/sanitizer_synccheck_nostash.txt; tail -3 $R/sanitizer_synccheck_nostash.txt
