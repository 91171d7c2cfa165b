mkdir -p gpurun_out/r01
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > gpurun_out/r01/sanitizer_$tool.txt 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/r01/sanitizer_$tool.txt
done
