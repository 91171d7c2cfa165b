mkdir -p gpurun_out/r01
SKIP_STRATS=thread timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_run.py > gpurun_out/r01/sanitizer_synccheck_nothread.txt 2>&1
echo "rc=$?"; tail -3 gpurun_out/r01/sanitizer_synccheck_nothread.txt
