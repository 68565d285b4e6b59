#!/bin/bash
# One gpurun call: smoke + the default bench line (+ detail) into gpurun_out/.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke_rc=$?" >> gpurun_out/smoke.log
timeout 1500 python bench.py ${BENCH_ARGS} --detail gpurun_out/bench_detail.json > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench_rc=$?" >> gpurun_out/bench.err
tail -c 2500 gpurun_out/bench.json | tail -n1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("PARSED", len(json.dumps(d)), d["value"], d.get("speedup_geomean"))' >> gpurun_out/bench.err 2>&1
tail -n 5 gpurun_out/smoke.log gpurun_out/bench.err
