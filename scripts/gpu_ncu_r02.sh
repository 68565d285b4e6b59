#!/bin/bash
# ncu evidence for round 2 (one GPU), into gpurun_out/:
#  1. metric pass: every benched member + fused kernel (DL and crypto) -> ncu_r02.csv + order
#  2. launch list of the bench's timed step (NVTX range "step")        -> launches_r02.csv
#  3. --set full of the dominant fused kernel                          -> prof_dom_r02.ncu-rep
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,smsp__inst_executed.sum,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__block_size
timeout 1200 ncu --metrics $M --clock-control none -k regex:'^(bn_|hist|im2col|maxpool|upsample|fused|sha256d|blake|ethash)' --csv --log-file gpurun_out/ncu_r02.csv python scripts/ncu_launch_r02.py --finalists > gpurun_out/ncu_r02.order 2> gpurun_out/ncu_r02.err
echo "metrics_rc=$?" >> gpurun_out/ncu_r02.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "step/" \
  --csv --log-file gpurun_out/launches_r02.csv python bench.py --steps 3 --warmup 3 --no-crypto --no-cpu-baseline --no-parity --no-ceilings --detail gpurun_out/launch_bench_detail.json \
  > gpurun_out/launches_r02.log 2>&1
echo "launches_rc=$?" >> gpurun_out/launches_r02.log
DOM=$(python -c "import json;d=json.load(open('profiles/r02_bench_line.json'));print(d['roofline']['kernel'].split()[-1])")
K=$(python -c "a,b='$DOM'.split('+'); n={'bn':'bn_stats'}; print('fused_'+n.get(a,a)+'_'+n.get(b,b))")
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^$K" -c 1 -o gpurun_out/prof_dom_r02 -f python scripts/ncu_launch_r02.py --only $DOM --fused-only --no-crypto >> gpurun_out/ncu_r02.err 2>&1
echo "full_rc=$? dom=$DOM kernel=$K" >> gpurun_out/ncu_r02.err
