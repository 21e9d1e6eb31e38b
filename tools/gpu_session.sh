mkdir -p gpurun_out/sanitize
timeout 300 python tools/sanitize_run.py 2>&1 | tail -3
for tool in memcheck racecheck synccheck initcheck; do
  start=$(date +%s)
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 99 python tools/sanitize_run.py > gpurun_out/sanitize/${tool}_default.log 2>&1
  rc=$?
  echo "$tool rc=$rc $(( $(date +%s) - start ))s $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|all checks passed|FAILURES' gpurun_out/sanitize/${tool}_default.log | tr '\n' ' ')"
done
