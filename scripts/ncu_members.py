"""Launch every member unfused and selected fused pairs once each (for ncu captures).
python scripts/ncu_members.py [--grid 296] [--pairs bn+hist:640,bn+upsample:384]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
from paper_2007_01277_b200 import hfuse as hf  # noqa: E402
from paper_2007_01277_b200 import pairs as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--grid", type=int, default=296)
ap.add_argument("--members", default=",".join(P.ORDER))
ap.add_argument("--pairs", default="")
ap.add_argument("--form", default="b200")
args = ap.parse_args()
keys = [k for k in args.members.split(",") if k]
pairs = [p.split(":") for p in args.pairs.split(",") if p]
need = sorted(set(keys) | {k for p, _ in pairs for k in p.split("+")})
img = hf.Image(P.MEMBERS[need[0]].sizes["full"](0).image)
for k in need[1:]:
    img.merge(hf.Image(P.MEMBERS[k].sizes["full"](0).image))
img.upload()
for k in keys:
    hf.Module.kernel(P.source(args.form, P.MEMBERS[k].stem), grid=args.grid, specialize=img).run(img, args.grid)
for p, d1 in pairs:
    a, b = p.split("+")
    m = hf.Module.fused(P.source(args.form, P.MEMBERS[a].stem), P.source(args.form, P.MEMBERS[b].stem),
                        int(d1), 1024 - int(d1), grid=args.grid, specialize=img)
    m.run(img, args.grid)
import ctypes  # noqa: E402
ctypes.CDLL("libcudart.so.12").cudaDeviceSynchronize()
print("done")
