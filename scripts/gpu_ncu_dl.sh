#!/bin/bash
# ncu evidence for the DL members and fused pairs at the bench's configurations (one GPU):
#  1. metric pass over every member + fused pair  -> gpurun_out/ncu_dl.csv (traffic, issue, stalls)
#  2. --set full of the dominant fused kernel      -> gpurun_out/prof_dom.ncu-rep
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
B=profiles/r01_bench_full.json
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,smsp__inst_executed.sum,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__block_size,l1tex__throughput.avg.pct_of_peak_sustained_active,lts__throughput.avg.pct_of_peak_sustained_elapsed
timeout 900 ncu --metrics $M --clock-control none -k regex:'^(bn_|hist|im2col|maxpool|upsample|fused)' --csv --log-file gpurun_out/ncu_dl.csv python scripts/ncu_members.py --from-bench $B > gpurun_out/ncu_dl.log 2>&1
echo "metrics_rc=$?" >> gpurun_out/ncu_dl.log
DOM=$(python -c "import json;d=json.loads(open('$B').read().strip().splitlines()[-1]);print(d['roofline']['kernel'].split()[-1])")
K=$(python -c "a,b='$DOM'.split('+'); n={'bn':'bn_stats'}; print('fused_'+n.get(a,a)+'_'+n.get(b,b))")
echo "dominant $DOM kernel $K" >> gpurun_out/ncu_dl.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^$K" -c 1 -o gpurun_out/prof_dom -f python scripts/ncu_members.py --from-bench $B --only-pairs $DOM >> gpurun_out/ncu_dl.log 2>&1
echo "full_rc=$?" >> gpurun_out/ncu_dl.log
