#!/bin/bash
# One gpurun call: the binding test, ncu refresh, conv3 shapes and the reference arm.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_binding_gpu.py tests/test_runtime_gpu.py -q > gpurun_out/t_extra.log 2>&1
bash scripts/gpu_ncu_r02.sh
timeout 1500 python bench.py --shapes conv3 --no-crypto --detail gpurun_out/bench_conv3_detail.json > gpurun_out/bench_conv3.json 2> gpurun_out/bench_conv3.err
(time timeout 1500 python bench.py --impl reference) > gpurun_out/ref.json 2> gpurun_out/ref.err
true
