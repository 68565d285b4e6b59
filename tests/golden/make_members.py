"""Member / pair fixtures from the UNMODIFIED reference interpreter (TEST INFRASTRUCTURE).

For every DL member (paper_2007_01277_b200/pairs.py) at the `tiny` and `parity` sizes:
  ref   : run_functional of the naive form kernels/ref/<stem>.mk
  b200  : run_functional of the B200 form after `hfuse lower` (MK+ -> Mini-Kernel)
recording the FNV-1a digest and the output arrays (float32 as raw bits). For every pair
at the parity size and d1 in SPLITS: the reference's sequential run (k1 at d1 threads,
then k2 at d2) of the lowered B200 forms, which the fused sm_100a kernel must reproduce
bit for bit. All runs use grid GRID. Written to members.json.
"""
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

GRID = 4
SPLITS = [256, 512, 768]
BN_GRIDS = [3, 7, 16, 37]
WARP_SLOTS = 256  # >= (37 / 8 + 2) * 32
RAGGED = [1, 3, 1001, 4099]
OUTPUTS = {"bn": ["bn_stats"], "hist": ["hi_out"], "maxpool": ["mp_y", "mp_idx"], "upsample": ["us_y"],
           "im2col": ["ic_col"]}


def bits(a):
    import numpy as np
    return [int(v) for v in np.asarray(a).view(np.uint32)]


def main():
    out = {"grid": GRID, "splits": SPLITS, "members": {}, "pairs": {}}
    with tempfile.TemporaryDirectory() as d:
        lowered = {}
        for key, m in pairs.MEMBERS.items():
            p = os.path.join(d, f"{m.stem}_b200.mk")
            with open(p, "w") as f:
                f.write(hf.lower(pairs.source("b200", m.stem)))
            lowered[key] = p
        for key, m in pairs.MEMBERS.items():
            rec = {}
            for size in ("tiny", "parity"):
                img = os.path.join(d, f"{key}_{size}.img")
                with open(img, "w") as f:
                    f.write(m.sizes[size](0).image)
                row = {}
                for form, path in (("ref", os.path.join(pairs.KERNELS, "ref", m.stem + ".mk")), ("b200", lowered[key])):
                    dig, secs, dump = oracle.ref_run("run", path, "--mem", img, "--grid", GRID)
                    arrays, _ = oracle.parse_image(dump)
                    row[form] = {"digest": dig, "outputs": {n: bits(arrays[n]) for n in OUTPUTS[key]}}
                rec[size] = row
            out["members"][key] = rec
        for a, b in pairs.PAIRS:
            ma, mb = pairs.MEMBERS[a], pairs.MEMBERS[b]
            img = os.path.join(d, f"{a}_{b}.img")
            with open(img, "w") as f:
                f.write(ma.sizes["parity"](0).image + mb.sizes["parity"](0).image)
            row = {}
            for d1 in SPLITS:
                dig, _, dump = oracle.ref_run("seq", lowered[a], lowered[b], "--d1", d1, "--d2", 1024 - d1, "--mem", img,
                                              "--grid", GRID)
                arrays, _ = oracle.parse_image(dump)
                row[str(d1)] = {"digest": dig,
                                "outputs": {n: bits(arrays[n]) for n in OUTPUTS[a] + OUTPUTS[b]}}
            out["pairs"][f"{a}+{b}"] = row
        # the grid-balanced BatchNorm variant at grids where channels straddle blocks (and, at
        # tiny size with grid 16 > its 12 vectors, where some blocks own no vectors)
        bal = os.path.join(d, "batchnorm_balanced_b200.mk")
        with open(bal, "w") as f:
            f.write(hf.lower(pairs.source("b200", "batchnorm_balanced")))
        with open(os.path.join(d, "hist_ref.mk"), "w") as f:
            f.write(pairs.source("ref", "histogram"))
        out["bn_grids"] = {}
        for size in ("tiny", "parity"):
            img = os.path.join(d, f"bn_{size}_grids.img")
            with open(img, "w") as f:
                f.write(pairs.MEMBERS["bn"].sizes[size](0).image)
            out["bn_grids"][size] = {}
            for g in BN_GRIDS:
                dig, _, _ = oracle.ref_run("run", bal, "--mem", img, "--grid", g)
                out["bn_grids"][size][str(g)] = dig
        # warp-level hand-off form (atomic_add_release / load_relaxed): WARP_SLOTS partial slots
        warp = os.path.join(d, "bn_warp.mk")
        with open(warp, "w") as f:
            f.write(hf.lower(pairs.source("b200", "batchnorm_warp")))
        out["bn_warp_grids"] = {}
        for size, dims in (("tiny", (1, 3, 16)), ("parity", (2, 8, 56 * 56))):
            img = os.path.join(d, f"bn_{size}_warp.img")
            with open(img, "w") as f:
                f.write(pairs._bn(*dims, slots=WARP_SLOTS)(0).image)
            out["bn_warp_grids"][size] = {}
            for g in BN_GRIDS:
                dig, _, _ = oracle.ref_run("run", warp, "--mem", img, "--grid", g)
                out["bn_warp_grids"][size][str(g)] = dig
        # ragged histogram lengths (n % 4 != 0, n < 4): the reference form and the B200 form
        out["hist_ragged"] = {}
        for n in RAGGED:
            img = os.path.join(d, f"hist_{n}.img")
            with open(img, "w") as f:
                f.write(pairs._hist(n, -4.5, 4.5)(0).image)
            for g in (4, 37):
                dig_ref, _, _ = oracle.ref_run("run", os.path.join(d, "hist_ref.mk"), "--mem", img, "--grid", g)
                dig_b200, _, _ = oracle.ref_run("run", lowered["hist"], "--mem", img, "--grid", g)
                assert dig_ref == dig_b200, (n, g)
                out["hist_ragged"][f"{n}/{g}"] = dig_b200
    with open(os.path.join(HERE, "members.json"), "w") as f:
        json.dump(out, f, sort_keys=True)
    print("members fixtures written")


if __name__ == "__main__":
    main()
