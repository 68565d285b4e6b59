"""Launch every member unfused and selected fused pairs once each (for ncu captures).
python scripts/ncu_members.py [--grid 296] [--pairs bn+hist:640,bn+upsample:384]
python scripts/ncu_members.py --from-bench profiles/r01_bench_full.json [--only-pairs bn+hist,...]
  (every member at its bench grid, every fused pair at the bench's (grid, split, cap); all
  modules JIT-specialized to the image exactly as bench.py builds them)"""
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
ap.add_argument("--from-bench", default="")
ap.add_argument("--only-pairs", default="")
args = ap.parse_args()
keys = [k for k in args.members.split(",") if k]
pairs = [p.split(":") for p in args.pairs.split(",") if p]
bench = None
if args.from_bench:
    import json
    bench = json.loads(open(args.from_bench).read().strip().splitlines()[-1])
    rows = bench["pairs"]
    if args.only_pairs:
        rows = [r for r in rows if r["pair"] in args.only_pairs.split(",")]
        keys = []
    pairs = [(r["pair"], r["d1"], r["grid"], r["reg_cap"], r["d2"]) for r in rows]
    mgrid = {}
    for r in bench["pairs"]:
        a, b = r["pair"].split("+")
        mgrid[a], mgrid[b] = r["grid_a"], r["grid_b"]
need = sorted(set(keys) | {k for p in pairs for k in p[0].split("+")})
img = hf.Image(P.MEMBERS[need[0]].sizes["full"](0).image)
for k in need[1:]:
    img.merge(hf.Image(P.MEMBERS[k].sizes["full"](0).image))
img.upload()
for k in keys:
    g = mgrid[k] if bench else args.grid
    hf.Module.kernel(P.source(args.form, P.MEMBERS[k].stem), grid=g, specialize=img).run(img, g)
for p in pairs:
    a, b = p[0].split("+")
    g = int(p[2]) if len(p) > 2 else args.grid
    cap = p[3] if len(p) > 3 and p[3] else "off"
    d2 = int(p[4]) if len(p) > 4 else 1024 - int(p[1])
    m = hf.Module.fused(P.source(args.form, P.MEMBERS[a].stem), P.source(args.form, P.MEMBERS[b].stem),
                        int(p[1]), d2, regcap=cap, grid=g, specialize=img)
    m.run(img, g)
import ctypes  # noqa: E402
ctypes.CDLL("libcudart.so.12").cudaDeviceSynchronize()
print("done")
