"""Launch one member / fused kernel a few times for ncu (never a bench number).

python scripts/ncu_target.py bn hist --d1 512 [--form b200] [--only a|b|fused] [--grid G]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
from paper_2007_01277_b200 import hfuse as hf  # noqa: E402
from paper_2007_01277_b200.pairs import MEMBERS, source  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("a")
ap.add_argument("b")
ap.add_argument("--d1", type=int, default=512)
ap.add_argument("--d0", type=int, default=1024)
ap.add_argument("--form", default="b200")
ap.add_argument("--only", default="all")
ap.add_argument("--grid", type=int, default=0)
ap.add_argument("--regcap", default="off")
ap.add_argument("--launches", type=int, default=2)
args = ap.parse_args()
ma, mb = MEMBERS[args.a], MEMBERS[args.b]
img = hf.Image(ma.sizes["full"](0).image).merge(hf.Image(mb.sizes["full"](0).image)).upload()
sa, sb = source(args.form, ma.stem), source(args.form, mb.stem)
mods = []
if args.only in ("all", "a"):
    mods.append(hf.Module.kernel(sa, grid=args.grid))
if args.only in ("all", "b"):
    mods.append(hf.Module.kernel(sb, grid=args.grid))
if args.only in ("all", "fused"):
    mods.append(hf.Module.fused(sa, sb, args.d1, args.d0 - args.d1, regcap=args.regcap, grid=args.grid))
for m in mods:
    for _ in range(args.launches):
        m.run(img, args.grid)
import ctypes  # noqa: E402
ctypes.CDLL("libcudart.so.12").cudaDeviceSynchronize()
print("launched", [m.entry for m in mods])
