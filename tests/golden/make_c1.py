"""C1 / C2 at full size on the UNMODIFIED reference interpreter (TEST INFRASTRUCTURE; BASELINE
configs[0]: BatchNorm-collect-stats + Hist on a 64x256x56x56 fp32 tensor, equivalence check; and
the other nine DL pairs at their C2 sizes).
The B200 member forms, lowered to plain Mini-Kernel (hfuse lower), run sequentially at the split
d1/d2 and grid G the GPU test fuses them with (run_functional, acceptance_main.cpp:147-152); the
fused sm_100a kernel must reproduce the resulting FNV-1a digest over all arrays bit for bit.
Writes c1_full.json (BN + Hist) and full_pairs.json (all ten pairs): digest, split, grid, the
interpreter's wall time. `python tests/golden/make_c1.py [--pairs]` (the ten pairs take minutes)."""
import json
import os
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.abspath(os.path.join(HERE, "..", ".."))
sys.path.insert(0, ROOT)

from oracle import oracle  # noqa: E402
from paper_2007_01277_b200 import hfuse as hf  # noqa: E402
from paper_2007_01277_b200 import pairs  # noqa: E402

D1, D2, GRID = 512, 512, 296


def run_pair(a, b):
    ma, mb = pairs.MEMBERS[a], pairs.MEMBERS[b]
    with tempfile.TemporaryDirectory() as d:
        k1, k2, img = (os.path.join(d, n) for n in ("k1.mk", "k2.mk", "pair.img"))
        open(k1, "w").write(hf.lower(pairs.source("b200", ma.stem)))
        open(k2, "w").write(hf.lower(pairs.source("b200", mb.stem)))
        open(img, "w").write(ma.sizes["full"](0).image + mb.sizes["full"](0).image)
        r = subprocess.run([oracle.REF, "seq", k1, k2, "--d1", str(D1), "--d2", str(D2), "--mem", img, "--grid",
                            str(GRID), "--time"], capture_output=True, text=True, timeout=3600)
        if r.returncode != 0:
            raise RuntimeError(r.stderr)
        kv = dict(line.split(" = ") for line in r.stdout.strip().splitlines())
    return {"pair": f"{a}+{b}", "form": "b200 (lowered)", "d1": D1, "d2": D2, "grid": GRID,
            "digest": kv["digest"], "interpreter_seconds": float(kv["seconds"])}


def main():
    out = run_pair("bn", "hist")
    json.dump(out, open(os.path.join(HERE, "c1_full.json"), "w"), indent=1)
    print(json.dumps(out), flush=True)
    if "--pairs" in sys.argv:
        allp = {}
        for a, b in pairs.PAIRS:
            allp[f"{a}+{b}"] = out if (a, b) == ("bn", "hist") else run_pair(a, b)
            print(json.dumps(allp[f"{a}+{b}"]), flush=True)
        json.dump(allp, open(os.path.join(HERE, "full_pairs.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
