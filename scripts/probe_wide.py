"""Probe: a much wider fused-configuration sweep for the DL pairs that lose to two-stream at C2
(d0 in {384..1024} step 128, 32-thread splits, grids 148 x {1..32}, caps none/r0/32/40/48),
top-5 points re-timed against the two-stream baseline at its best grid pair. Graph protocol.
JSON lines on stdout."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2007_01277_b200 import hfuse as hf  # noqa: E402
from paper_2007_01277_b200 import pairs as P  # noqa: E402

pairs = [tuple(p.split("+")) for p in (sys.argv[1] if len(sys.argv) > 1 else
                                      "bn+im2col,bn+upsample,im2col+upsample,maxpool+upsample").split(",")]
GRIDS = [148 * k for k in (1, 2, 4, 8, 16, 24, 32)]
import torch  # noqa: E402
stream = torch.cuda.current_stream()
for a, b in pairs:
    wa, wb = P.MEMBERS[a].sizes["full"](), P.MEMBERS[b].sizes["full"]()
    img = hf.Image(wa.image).merge(hf.Image(wb.image)).upload(stream)
    sa, sb = P.source("b200", P.MEMBERS[a].stem), P.source("b200", P.MEMBERS[b].stem)
    ka, kb = hf.Module.kernel(sa, grid=296, specialize=img), hf.Module.kernel(sb, grid=296, specialize=img)
    screen = {(x, y): hf.time_graph("two_stream", ka, kb, img, x, y, reps=5, samples=3)["mean_us"]
              for x in GRIDS for y in GRIDS}
    tx, ty = min(screen, key=screen.get)
    two = hf.time_graph("two_stream", ka, kb, img, tx, ty, reps=20, samples=5)
    pts = []
    for d0 in (384, 512, 640, 768, 896, 1024):
        for g in GRIDS:
            try:
                r = hf.search(sa, sb, img, d0=d0, grid=g, reps=5, warmup=1, specialize=True, flush_l2=False,
                              granularity=32, extra_caps=(32, 40, 48))
            except hf.HFuseError as e:
                print(json.dumps({"pair": f"{a}+{b}", "d0": d0, "grid": g, "err": str(e)[:120]}), flush=True)
                continue
            pts += [(t["us"], d0, g, t["d1"], t["reg_cap"]) for t in r["trace"]]
        print(json.dumps({"pair": f"{a}+{b}", "d0": d0, "points": len(pts),
                          "best_so_far": min(pts)[0] if pts else None}), flush=True)
    top = []
    for us, d0, g, d1, cap in sorted(pts)[:5]:
        c = None if cap in ("none", None) else int(cap)
        m = hf.Module.fused(sa, sb, d1, d0 - d1, regcap=c if c else "off", grid=g, specialize=img)
        t = hf.time_graph("single", m, None, img, g, 0, reps=20, samples=5)
        top.append({"d0": d0, "grid": g, "d1": d1, "cap": c, "screen_us": us, "us": round(t["mean_us"], 2),
                    "ci95": round(t["ci95_us"], 2)})
        del m
    best = min(top, key=lambda x: x["us"])
    print(json.dumps({"pair": f"{a}+{b}", "two_stream_us": round(two["mean_us"], 2), "two_grids": [tx, ty],
                      "best": best, "speedup": round(two["mean_us"] / best["us"], 4), "top": top,
                      "n_points": len(pts)}), flush=True)
    del img, ka, kb
