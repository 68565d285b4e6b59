"""Probe: the BatchNorm pairs' heterogeneous partition with fewer fused blocks than channels
(B1 < C: each fused block walks several channels) vs B1 = C. Graph protocol. JSON lines."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2007_01277_b200 import hfuse as hf  # noqa: E402
from paper_2007_01277_b200 import pairs as P  # noqa: E402

for b in ("im2col", "upsample", "maxpool"):
    wa, wb = P.MEMBERS["bn"].sizes["full"](), P.MEMBERS[b].sizes["full"]()
    img = hf.Image(wa.image).merge(hf.Image(wb.image)).upload()
    sa, sb = P.source("b200", "batchnorm"), P.source("b200", P.MEMBERS[b].stem)
    ka, kb = hf.Module.kernel(sa, grid=296, specialize=img), hf.Module.kernel(sb, grid=296, specialize=img)
    two = min(hf.time_graph("two_stream", ka, kb, img, x, y, reps=20, samples=5)["mean_us"]
              for x in (296, 592, 2368) for y in (296, 1184, 2368))
    rows = []
    for d0, d2 in ((1024, 128), (1024, 256), (768, 256), (512, 128), (512, 64)):
        for b1 in (64, 128, 192, 256):
            for cap in ("off", 32):
                m = hf.Module.fused_opts(sa, sb, d0 - d2, d2, regcap=cap, split_grid=b1, grid=b1, specialize=img)
                res = 148 * (2048 // d0)
                for g in sorted({b1 + res, 2 * res, 4 * res, 8 * res, 16 * res}):
                    if g < b1:
                        continue
                    t = hf.time_graph("single", m, None, img, g, 0, reps=10, samples=3)["mean_us"]
                    rows.append({"d0": d0, "d2": d2, "b1": b1, "cap": cap, "grid": g, "us": round(t, 2)})
    rows.sort(key=lambda r: r["us"])
    best_b1 = {}
    for r in rows:
        best_b1.setdefault(r["b1"], r)
    print(json.dumps({"pair": f"bn+{b}", "two_stream_us": round(two, 2), "best_per_b1": best_b1}), flush=True)
    del img, ka, kb
