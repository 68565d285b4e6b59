"""SASS of the lean Ethash seed hand-off (profiles/r02_ethash_seed_handoff_sass.txt): the 8-lane
groups exchange Keccak-512 seeds through shared memory, ordered in the source by MK+ warp_sync
(__syncwarp). ptxas compiles that sync to a divergence check (BRA.DIV) with no WARPSYNC on the
converged path between the seed STS and the partners' LDS. Context for the one racecheck report on
a degenerate launch shape (profiles/r02_racecheck_ethash_shapes.log). Runs on the CPU (NVRTC
source + nvcc -cubin).
python scripts/sass_ethash_handoff.py"""
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2007_01277_b200 import crypto as CR  # noqa: E402
from paper_2007_01277_b200 import hfuse as hf  # noqa: E402
from paper_2007_01277_b200 import pairs as P  # noqa: E402

img = hf.Image(CR.workload("ethash", 64, 2, nonce0=3, target=1 << 28).image)
m = hf.Module.kernel(open(os.path.join(P.KERNELS, "b200", "ethash.mk")).read(), grid=2, specialize=img)
src = m.source
lines = src.splitlines()
sync_line = next(i for i, l in enumerate(lines) if "__syncwarp();" in l) + 1
with tempfile.TemporaryDirectory() as d:
    cu, cubin = os.path.join(d, "ethash.cu"), os.path.join(d, "ethash.cubin")
    open(cu, "w").write(src)
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-cubin", "-lineinfo", "-o", cubin, cu],
                   check=True)
    sass = subprocess.run(["cuobjdump", "-sass", cubin], capture_output=True, text=True, check=True).stdout
ins = [l.strip() for l in sass.splitlines() if re.match(r"\s+/\*[0-9a-f]{4}\*/", l)]
first_sts = next(i for i, l in enumerate(ins) if "STS" in l)
first_lds = next(i for i, l in enumerate(ins) if "LDS" in l and i > first_sts)
window = ins[first_sts:first_lds + 12]
between = ins[first_sts:first_lds]
out = [__doc__.split("\npython")[0], "",
       f"source: __syncwarp() at line {sync_line} of the specialized ethash source (grid 2, 1,024 threads)",
       f"WARPSYNC between the first seed STS and the first partner LDS: {any('WARPSYNC' in l for l in between)}",
       f"WARPSYNC anywhere in the kernel: {sum('WARPSYNC' in l for l in ins)} (warp_bcast's partial-warp path)", ""]
out += window
path = os.path.join(ROOT, "profiles", "r02_ethash_seed_handoff_sass.txt")
open(path, "w").write("\n".join(out) + "\n")
print("\n".join(out[:6]))
