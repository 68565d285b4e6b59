#!/bin/bash
# One gpurun call after scripts/gpu_round.sh (its bench line/detail copied to profiles/): the ncu
# refresh at the benched configurations, the C5 conv3_x shapes, rank 0's 1/8 share on one GPU
# (the per-GPU figure of an 8-GPU strong-scaling job) and the reference arm. Into gpurun_out/.
mkdir -p gpurun_out
bash scripts/gpu_ncu_r02.sh > gpurun_out/ncu_run.txt 2>&1
timeout 1500 python bench.py --shapes conv3 --no-crypto --detail gpurun_out/bench_conv3_detail.json > gpurun_out/bench_conv3.json 2> gpurun_out/bench_conv3.err
timeout 1500 python bench.py --shard-of 8 --no-crypto --detail gpurun_out/bench_shard8_detail.json > gpurun_out/bench_shard8.json 2> gpurun_out/bench_shard8.err
(time timeout 1500 python bench.py --impl reference) > gpurun_out/ref.json 2> gpurun_out/ref.err
rm -f gpurun_out/sanitize_summary.txt; bash scripts/gpu_sanitize.sh > gpurun_out/sanitize_out.txt 2>&1
tail -n1 gpurun_out/bench_conv3.json gpurun_out/bench_shard8.json gpurun_out/ref.json | cut -c1-400
true
