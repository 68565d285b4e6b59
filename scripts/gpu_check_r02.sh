#!/bin/bash
# One gpurun call: racecheck of the Ethash forms alone (full output), the 1/8-share bench and the
# default bench line, into gpurun_out/.
mkdir -p gpurun_out
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python scripts/sanitize_targets.py ethash \
  > gpurun_out/racecheck_ethash.log 2>&1; echo "racecheck_ethash rc=$?" >> gpurun_out/racecheck_ethash.log
timeout 1500 python bench.py --shard-of 8 --no-crypto --detail gpurun_out/bench_shard8_detail.json > gpurun_out/bench_shard8.json 2> gpurun_out/bench_shard8.err
timeout 1700 python bench.py --detail gpurun_out/bench_detail.json > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench_rc=$?" >> gpurun_out/bench.err
tail -n 4 gpurun_out/racecheck_ethash.log; tail -c 300 gpurun_out/bench.json; true
