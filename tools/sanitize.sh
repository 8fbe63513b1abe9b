set -x
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_run.py > gpurun_out/sanitizer_$tool.log 2>&1; echo "$tool rc=$?"
  tail -4 gpurun_out/sanitizer_$tool.log
done
