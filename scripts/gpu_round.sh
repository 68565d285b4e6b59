#!/bin/bash
# One gpurun call: GPU tests + smoke, the 2-rank strong-scaling bench on one GPU (gloo), and the
# default 1-GPU bench line, all into gpurun_out/.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q ${PYTEST_ARGS} > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke_rc=$?" >> gpurun_out/smoke.log
if [ -z "$NO_TWO_RANK" ]; then
HF_BENCH_DIST=gloo timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 2 --steps 5 --warmup 3 --no-ceilings --detail gpurun_out/bench2_detail.json > gpurun_out/bench2.json 2> gpurun_out/bench2.err
echo "bench2_rc=$?" >> gpurun_out/bench2.err
fi
timeout 1500 python bench.py ${BENCH_ARGS} --detail gpurun_out/bench_detail.json > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench_rc=$?" >> gpurun_out/bench.err
tail -n 3 gpurun_out/gpu_tests.log gpurun_out/smoke.log gpurun_out/bench.err; true
