"""Probe: heterogeneous partitions with a one-warp member-2 interval in the fused blocks (d2 = 32:
the fused blocks are almost all member 1, member-2-only blocks are d0/32 one-warp sub-blocks),
the closest one launch gets to two concurrent launches. BN pairs, graph protocol. JSON lines."""
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
    two = min((hf.time_graph("two_stream", ka, kb, img, x, y, reps=20, samples=5)["mean_us"], x, y)
              for x in (296, 592, 2368) for y in (296, 1184, 2368, 4736))
    rows = []
    for d0 in (1024, 768, 512):
        for d2 in (32, 64, 128):
            for cap in ("off", 32):
                m = hf.Module.fused_opts(sa, sb, d0 - d2, d2, regcap=cap, split_grid=256, grid=256, specialize=img)
                res = 148 * (2048 // d0)
                for g in sorted({256 + res, 2 * res, 4 * res, 8 * res, 16 * res}):
                    if g < 256:
                        continue
                    t = hf.time_graph("single", m, None, img, g, 0, reps=10, samples=3)["mean_us"]
                    rows.append({"d0": d0, "d2": d2, "cap": cap, "grid": g, "us": round(t, 2)})
    rows.sort(key=lambda r: r["us"])
    print(json.dumps({"pair": f"bn+{b}", "two_stream": two, "top": rows[:6]}), flush=True)
    del img, ka, kb
