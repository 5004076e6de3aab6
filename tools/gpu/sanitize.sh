mkdir -p gpurun_out/sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 --log-file gpurun_out/sanitizer/$tool.log python tools/sanitize_run.py > gpurun_out/sanitizer/$tool.out 2>&1
  echo "$tool rc=$?"; tail -2 gpurun_out/sanitizer/$tool.log
done
