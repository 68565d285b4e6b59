#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over scripts/sanitize_targets.py (one GPU)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
    python scripts/sanitize_targets.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_summary.txt
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|hazard|sanitize targets" gpurun_out/sanitize_$tool.log | tail -n 4 >> gpurun_out/sanitize_summary.txt
done
cat gpurun_out/sanitize_summary.txt
