#!/bin/bash
# ncu metric pass over the crypto members and fused pairs (scripts/ncu_crypto.py), one GPU.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
M=gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,launch__registers_per_thread,smsp__inst_executed.sum,dram__bytes_read.sum,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,launch__occupancy_limit_registers,sm__maximum_warps_per_active_cycle_pct,sm__inst_executed_pipe_alu.sum,smsp__warps_issue_stalled_long_scoreboard.avg,smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio
timeout 900 ncu --metrics $M --clock-control none -k regex:'^(blake|ethash|sha|fused|upsample)' --csv --log-file gpurun_out/ncu_crypto.csv python scripts/ncu_crypto.py > gpurun_out/ncu_crypto.log 2>&1
echo "ncu_rc=$?" >> gpurun_out/ncu_crypto.log
