#!/bin/bash
# ncu launch list of the bench's timed step (the B200_PROFILING recipe's gpu__time_duration pass,
# restricted to the NVTX range "step": the K steps whose time is `value`), one GPU.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "step/" \
  --csv --log-file gpurun_out/launches_step.csv python bench.py --steps 3 --warmup 3 --no-crypto --no-cpu-baseline --ratios none \
  > gpurun_out/launches_step.log 2>&1
echo "ncu_rc=$?" >> gpurun_out/launches_step.log
grep -c '"gpu__time_duration.sum"' gpurun_out/launches_step.csv >> gpurun_out/launches_step.log
