"""Launch each crypto member once at the bench's C3 nonce counts (for the ncu instruction-count
pass that feeds the issue-rate roofline of the crypto pairs).

    ncu --metrics smsp__inst_executed.sum,sm__inst_executed_pipe_alu.sum,gpu__time_duration.sum,\
dram__bytes_read.sum --csv --log-file gpurun_out/crypto_inst.csv python scripts/ncu_crypto_inst.py
    python scripts/ncu_summarize.py crypto gpurun_out/crypto_inst.csv > profiles/crypto_inst.json
"""
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
from paper_2007_01277_b200 import crypto as CR  # noqa: E402
from paper_2007_01277_b200 import hfuse as hf  # noqa: E402
from paper_2007_01277_b200 import pairs as P  # noqa: E402

COUNTS = {"sha256d": 1 << 24, "blake2b": 1 << 23, "blake256": 1 << 24, "ethash": 1 << 20}
G = 296
for k, n in COUNTS.items():
    w = CR.workload(k, n, G, npages=1 << 25)
    img = hf.Image(w.image).upload()
    src = open(os.path.join(P.KERNELS, "b200", k + ".mk")).read()
    hf.Module.kernel(src, grid=G, specialize=img).run(img, G)
    del img
import ctypes  # noqa: E402
ctypes.CDLL("libcudart.so.12").cudaDeviceSynchronize()
print("done")
