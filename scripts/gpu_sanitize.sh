#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over scripts/sanitize_targets.py (one GPU).
# racecheck runs the Ethash forms alone in a separate process (`ethash`): one racecheck process
# over every target at once did not terminate cleanly (rc 11).
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for run in "memcheck:" "racecheck:no-ethash" "racecheck:ethash" "synccheck:"; do
  tool=${run%%:*}; arg=${run#*:}
  log=gpurun_out/sanitize_${tool}${arg:+_$arg}.log
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
    python scripts/sanitize_targets.py $arg > $log 2>&1
  echo "$tool ${arg:-all} rc=$?" >> gpurun_out/sanitize_summary.txt
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|hazard|Race reported|sanitize targets" $log | tail -n 4 >> gpurun_out/sanitize_summary.txt
done
cat gpurun_out/sanitize_summary.txt
