#!/bin/bash
# Round-end evidence in one call: crypto instruction counts (ncu; feeds the crypto roofline),
# GPU tests, smoke, and the default bench line.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 600 ncu --metrics smsp__inst_executed.sum,sm__inst_executed_pipe_alu.sum,gpu__time_duration.sum,dram__bytes_read.sum \
  --clock-control none --csv --log-file gpurun_out/crypto_inst.csv python scripts/ncu_crypto_inst.py > gpurun_out/crypto_inst.log 2>&1
python scripts/ncu_summarize.py crypto gpurun_out/crypto_inst.csv > gpurun_out/crypto_inst.json && cp gpurun_out/crypto_inst.json profiles/crypto_inst.json
bash scripts/gpu_verify.sh
