"""Probe: heterogeneous CTA partition (hf_build_fused_opts split_grid) vs the static fused
kernel and two-stream, at C2 sizes: blocks below B1 run both members, blocks above give all
threads to member 2 as d0/d2 sub-blocks. Graph protocol; best point oracle-checked. JSON lines."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2007_01277_b200 import hfuse as hf  # noqa: E402
from paper_2007_01277_b200 import pairs as P  # noqa: E402
from oracle import check as CK  # noqa: E402

detail = json.load(open(os.path.join(ROOT, "profiles", "r02_bench_detail.json")))
static = {r["pair"]: r for r in detail["results"]}
pairs = [tuple(p.split("+")) for p in (sys.argv[1] if len(sys.argv) > 1 else
                                      "bn+im2col,bn+upsample,bn+maxpool,im2col+upsample,maxpool+upsample,"
                                      "hist+im2col,hist+upsample,hist+maxpool,im2col+maxpool").split(",")]
for a, b in pairs:
    wa, wb = P.MEMBERS[a].sizes["full"](), P.MEMBERS[b].sizes["full"]()
    img = hf.Image(wa.image).merge(hf.Image(wb.image)).upload()
    sa, sb = P.source("b200", P.MEMBERS[a].stem), P.source("b200", P.MEMBERS[b].stem)
    st = static[f"{a}+{b}"]
    ms = hf.Module.fused(sa, sb, st["d1"], st["d2"], regcap=st["reg_cap"] or "off", grid=st["grid"], specialize=img)
    t_static = hf.time_graph("single", ms, None, img, st["grid"], 0, reps=20, samples=5)["mean_us"]
    ka, kb = hf.Module.kernel(sa, grid=296, specialize=img), hf.Module.kernel(sb, grid=296, specialize=img)
    ga, gb = st["two_stream_grids"]
    t_two = hf.time_graph("two_stream", ka, kb, img, ga, gb, reps=20, samples=5)["mean_us"]
    b1s = [256] if a == "bn" else [148, 296, 592, 1184]
    rows = []
    for d0 in (1024, 768, 512):
        for k in (2, 4, 8):
            d2 = d0 // k
            if d2 < 64 or d2 % 32:
                continue
            d1 = d0 - d2
            for cap in ("off", 32):
                try:
                    m = hf.Module.fused_opts(sa, sb, d1, d2, regcap=cap, split_grid=b1s[0], grid=296, specialize=img)
                except hf.HFuseError as e:
                    print(json.dumps({"pair": f"{a}+{b}", "d0": d0, "d2": d2, "err": str(e)[:160]}), flush=True)
                    continue
                for b1 in b1s:
                    if b1 != b1s[0]:
                        m = hf.Module.fused_opts(sa, sb, d1, d2, regcap=cap, split_grid=b1, grid=296, specialize=img)
                    res = 148 * (2048 // d0)
                    for g in sorted({max(b1, res), b1 + res, 2 * b1 + res, res * 4, res * 8, res * 16}):
                        if g < b1:
                            continue
                        t = hf.time_graph("single", m, None, img, g, 0, reps=5, samples=3)["mean_us"]
                        rows.append({"d0": d0, "d1": d1, "d2": d2, "cap": cap, "b1": b1, "grid": g, "us": round(t, 2)})
    rows.sort(key=lambda r: r["us"])
    best = None
    for r in rows[:4]:
        m = hf.Module.fused_opts(sa, sb, r["d1"], r["d2"], regcap=r["cap"], split_grid=r["b1"], grid=r["grid"],
                                 specialize=img)
        t = hf.time_graph("single", m, None, img, r["grid"], 0, reps=20, samples=5)["mean_us"]
        if best is None or t < best[1]:
            best = (r, t, m)
    r, t, m = best
    img.upload()
    m.run(img, r["grid"])
    img.download()
    par = {k: CK.check_member(k, img.array, CK.member_expected(k, w.image))["ok"] for k, w in ((a, wa), (b, wb))}
    print(json.dumps({"pair": f"{a}+{b}", "best": r, "us": round(t, 2), "static_us": round(t_static, 2),
                      "two_stream_us": round(t_two, 2), "vs_two": round(t_two / t, 4),
                      "vs_static": round(t_static / t, 4), "parity": par, "top": rows[:6]}), flush=True)
    del img, ms, ka, kb, m
