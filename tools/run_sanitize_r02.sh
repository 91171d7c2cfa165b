#!/bin/bash
# Round-2 sanitizers at HEAD: memcheck / racecheck / initcheck / synccheck on every
# kernel (tools/sanitize_run.py), plus the minimal tcgen05 synccheck repro.
cd /root/repo; R=gpurun_out/san02; mkdir -p $R
nvcc -gencode arch=compute_100a,code=sm_100a -o tools/tmem_synccheck_repro tools/tmem_synccheck_repro.cu
for v in 0 1 2 3; do
  for tool in memcheck racecheck synccheck; do
    echo "== variant $v, $tool" >> $R/tmem_repro.txt
    timeout 120 compute-sanitizer --tool $tool tools/tmem_synccheck_repro $v >> $R/tmem_repro.txt 2>&1
    echo "exit $?" >> $R/tmem_repro.txt
  done
done
for tool in memcheck racecheck initcheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > $R/sanitizer_$tool.txt 2>&1
  echo "exit $?" >> $R/sanitizer_$tool.txt
  tail -4 $R/sanitizer_$tool.txt
done
SKIP_STRATS=thread timeout 1500 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_run.py > $R/sanitizer_synccheck_nothread.txt 2>&1
echo "exit $?" >> $R/sanitizer_synccheck_nothread.txt
tail -3 $R/sanitizer_synccheck_nothread.txt
grep -E "^== |ERROR SUMMARY|variant|exit" $R/tmem_repro.txt
