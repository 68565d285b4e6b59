"""Fused block size d0 = 512 vs 1024 for the DL pairs (steady-state protocol, best grid)."""
import json
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
from paper_2007_01277_b200 import hfuse as hf  # noqa: E402
from paper_2007_01277_b200 import pairs as P  # noqa: E402

img = hf.Image(P.MEMBERS[P.ORDER[0]].sizes["full"](0).image)
for k in P.ORDER[1:]:
    img.merge(hf.Image(P.MEMBERS[k].sizes["full"](0).image))
img.upload()
src = {k: P.source("b200", P.MEMBERS[k].stem) for k in P.ORDER}
pairs = [tuple(p.split("+")) for p in os.environ.get("PAIRS", "bn+im2col,hist+maxpool,maxpool+upsample,bn+hist").split(",")]
out = {}
for a, b in pairs:
    row = {}
    for d0, grids in ((1024, (296, 592, 1184, 2368)), (512, (592, 1184, 2368, 4736))):
        best = None
        for g in grids:
            r = hf.search(src[a], src[b], img, d0=d0, grid=g, reps=5, warmup=2, specialize=True, granularity=64,
                          flush_l2=False)
            if best is None or r["best_time"] < best[0]:
                best = (r["best_time"], g, r["d1"], r["reg_cap"])
        t, g, d1, cap = best
        m = hf.Module.fused(src[a], src[b], d1, d0 - d1, regcap=cap or "off", grid=g, specialize=img)
        row[str(d0)] = {"grid": g, "d1": d1, "cap": cap,
                        "us": round(hf.time("single", m, None, img, g, warmup=2, reps=30, flush_l2=False)["iqm_us"], 2)}
    out[f"{a}+{b}"] = row
    print(a, b, json.dumps(row), flush=True)
json.dump(out, open("gpurun_out/probe_d0.json", "w"), indent=1)
