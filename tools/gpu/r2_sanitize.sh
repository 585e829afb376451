for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_small.py > gpurun_out/r2_sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/r2_sanitize_$tool.log
done
