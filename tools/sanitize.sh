#!/bin/bash
# compute-sanitizer over tools/sanitize_run.py (every kernel family, checked
# against the oracle) for the default build and every variant switch.
#   tools/sanitize.sh [tool ...]   (default: memcheck racecheck synccheck initcheck)
mkdir -p gpurun_out/sanitize
tools=${*:-memcheck racecheck synccheck initcheck}
variants="default CQG_NO_PRUNE=1 CQG_NO_GRAPH=1 CQG_NO_NDC_CODE=1 CQG_NO_CLUSTER_INIT=1 CQG_INIT_TILE_MIN=1000"
for tool in $tools; do
  for v in $variants; do
    env_set=""; [ "$v" != "default" ] && env_set="$v"
    log=gpurun_out/sanitize/${tool}_${v%%=*}.log
    env $env_set timeout 900 compute-sanitizer --tool $tool --error-exitcode 99 python tools/sanitize_run.py > $log 2>&1
    rc=$?
    echo "$tool $v rc=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|all checks passed|FAILURES' $log | tr '\n' ' ')"
  done
done
