"""Upsample store-pattern probe (diagnostic; the variants other than 'current' are not
correct upsampling): does the half-sector interleave of the two 128-bit stores per thread
(float4 2t and 2t+1) cost bandwidth compared with two warp-contiguous stores?"""
import json
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
from paper_2007_01277_b200 import hfuse as hf  # noqa: E402
from paper_2007_01277_b200 import pairs as P  # noqa: E402

# the per-thread-store form these variants rewrite (superseded: kernels/b200/upsample.mk)
cur = open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "upsample_v1.mk")).read()
variants = {
    "current": cur,
    "split_halves": cur.replace("vstore(us_y, 2 * t, y0, y1, y2, y3);", "vstore(us_y, t, y0, y1, y2, y3);")
                       .replace("vstore(us_y, 2 * t + 1, y4, y5, y6, y7);", "vstore(us_y, total + t, y4, y5, y6, y7);"),
    "one_store": cur.replace("vstore(us_y, 2 * t + 1, y4, y5, y6, y7);", ""),
}
w = P.MEMBERS["upsample"].sizes["full"](0)
img = hf.Image(w.image).upload()
for name, src in variants.items():
    for g in (296, 1184):
        m = hf.Module.kernel(src, grid=g, specialize=img)
        t = hf.time("single", m, None, img, g, warmup=2, reps=20)["iqm_us"]
        print(json.dumps({"variant": name, "grid": g, "us": round(t, 2), "regs": m.info.regs}), flush=True)
