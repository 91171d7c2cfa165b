#!/bin/bash
# One ncu --set full capture + summary + stall table.
# usage: tools/run_ncu_one.sh <name> <kernel-regex> <prof_one args...>
cd /root/repo; mkdir -p gpurun_out/ncu
name=$1; kre=$2; shift 2
ncu --set full --clock-control none --import-source on -k regex:$kre -s 1 -c 1 -o gpurun_out/ncu/$name -f \
  python tools/prof_one.py "$@" > gpurun_out/ncu/$name.log 2>&1
python tools/ncu_summary.py gpurun_out/ncu/$name.ncu-rep > gpurun_out/ncu/$name.summary.txt 2>&1
ncu -i gpurun_out/ncu/$name.ncu-rep --page source --csv > gpurun_out/ncu/$name.source.csv 2>/dev/null
python tools/ncu_stalls.py gpurun_out/ncu/$name.source.csv 30 >> gpurun_out/ncu/$name.summary.txt 2>&1
cat gpurun_out/ncu/$name.summary.txt
