"""Probe: the Hist member with K = 4 (kernels/b200/histogram.mk), 6 and 8 128-bit loads in flight
per thread at 1,024 / 768 / 512 threads (scripts/gen_hist.py): full-size bins vs the C oracle, alone
at five grids, then fused with MaxPool and BatchNorm under a d0 = 1024 split search over four grids
(top-3 re-timed). Graph protocol. JSON lines (profiles/r02_probe_hist_mlp.jsonl)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import numpy as np  # noqa: E402
from gen_hist import gen_hist  # noqa: E402
from oracle import oracle  # noqa: E402
from paper_2007_01277_b200 import hfuse as hf  # noqa: E402
from paper_2007_01277_b200 import pairs as P  # noqa: E402

wh = P.MEMBERS["hist"].sizes["full"](0)
arrays, _ = oracle.parse_image(wh.image)
want = oracle.hist(arrays["hi_x"])
variants = {(K, t): gen_hist(K, t) for K in (4, 6, 8) for t in (1024, 768, 512)}
img = hf.Image(wh.image).upload()
alone = {}
for (K, t), src in variants.items():
    try:
        k = hf.Module.kernel(src, grid=296, specialize=img)
    except hf.HFuseError as e:
        print(json.dumps({"K": K, "threads": t, "error": str(e)[:200]}), flush=True)
        continue
    img.set_array("hi_out", np.zeros(64, np.int32))
    img.upload()
    k.run(img, 296)
    img.download()
    ok = bool(np.array_equal(img.array("hi_out"), want))
    ts = {g: round(hf.time_graph("single", k, None, img, g, 0, reps=10, samples=5)["mean_us"], 2)
          for g in (148, 296, 592, 1184, 2368)}
    alone[(K, t)] = min(ts.values())
    print(json.dumps({"K": K, "threads": t, "parity": ok, "regs": k.info.regs, "bps": k.info.blocks_per_sm,
                      "alone_us": ts}), flush=True)
    del k
best_forms = sorted(alone, key=alone.get)[:2]
forms = [(4, 1024)] + [f for f in best_forms if f != (4, 1024)]
for partner in ("maxpool", "bn"):
    wp = P.MEMBERS[partner].sizes["full"](0)
    im = hf.Image(wh.image).merge(hf.Image(wp.image)).upload()
    sp = P.source("b200", P.MEMBERS[partner].stem)
    for f in forms:
        sa, sb = (variants[f], sp) if partner == "maxpool" else (sp, variants[f])
        trace = []
        for g in (592, 1184, 2368, 4736):
            try:
                r = hf.search(sa, sb, im, d0=1024, grid=g, reps=5, warmup=1, specialize=True, flush_l2=False,
                              granularity=64)
            except hf.HFuseError:
                continue
            trace += [(g, t["d1"], t["reg_cap"], t["us"]) for t in r["trace"]]
        best = None
        for g, d1, cap, us in sorted(trace, key=lambda t: t[3])[:3]:
            cfg = {"d1": d1, "d2": 1024 - d1, "grid": g, "interval_regs": None,
                   "reg_cap": None if cap in ("none", None) else int(cap)}
            m = hf.Module.from_config(sa, sb, cfg, specialize=im)
            t = hf.time_graph("single", m, None, im, g, 0, reps=20, samples=7)["mean_us"]
            if best is None or t < best[1]:
                best = (cfg, t)
            del m
        pair = "hist+maxpool" if partner == "maxpool" else "bn+hist"
        print(json.dumps({"pair": pair, "K": f[0], "threads": f[1], "cfg": best[0], "fused_us": round(best[1], 2)}),
              flush=True)
    del im
