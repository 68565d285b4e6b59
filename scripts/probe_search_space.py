"""Wider DL search space: d0 in {512, 768, 1024} x 32-thread granularity vs the bench's
{512, 1024} x 64 -- does the finer/wider sweep find faster fused kernels? (steady-state timing)"""
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
GR = {1024: (296, 592, 1184, 2368), 768: (296, 592, 1184, 2368), 512: (592, 1184, 2368, 4736)}
out = {}
for a, b in P.PAIRS:
    row = {}
    for label, d0s, gran in (("bench", (1024, 512), 64), ("wide", (1024, 768, 512), 32)):
        best = None
        n = 0
        for d0 in d0s:
            for g in GR[d0]:
                r = hf.search(src[a], src[b], img, d0=d0, grid=g, reps=5, warmup=2, specialize=True,
                              granularity=gran, flush_l2=False)
                n += len(r["trace"])
                if best is None or r["best_time"] < best[0]:
                    best = (r["best_time"], d0, g, r["d1"], r["reg_cap"])
        t, d0, g, d1, cap = best
        m = hf.Module.fused(src[a], src[b], d1, d0 - d1, regcap=cap or "off", grid=g, specialize=img)
        us = hf.time("single", m, None, img, g, warmup=5, reps=60, flush_l2=False)["iqm_us"]
        row[label] = {"d0": d0, "grid": g, "d1": d1, "cap": cap, "us": round(us, 2), "points": n}
    out[f"{a}+{b}"] = row
    print(a, b, json.dumps(row), flush=True)
json.dump(out, open("gpurun_out/probe_search_space.json", "w"), indent=1)
