"""Probe: BatchNorm statistics with K 128-bit loads in flight per thread (scripts/gen_bn.py) at
several block sizes, alone (graph protocol, parity vs fp64) and fused with Hist / Im2Col under the
bench's own search (bench.search_pair). JSON lines on stdout (profiles/r02_probe_bn_mlp.jsonl)."""
import json
import os
import sys
import types

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import gen_bn  # noqa: E402
from oracle import check as CK  # noqa: E402
from paper_2007_01277_b200 import hfuse as hf  # noqa: E402
from paper_2007_01277_b200 import pairs as P  # noqa: E402

variants = [(4, 1024), (6, 1024), (8, 1024), (8, 768), (8, 512), (6, 768), (12, 512)]
wa = P.MEMBERS["bn"].sizes["full"]()
img = hf.Image(wa.image).upload()
x = None
res = {}
for K, T in variants:
    src = gen_bn.gen_bn(K, T)
    try:
        k = hf.Module.kernel(src, grid=296, specialize=img)
    except hf.HFuseError as e:
        print(json.dumps({"K": K, "threads": T, "err": str(e)[:200]}), flush=True)
        continue
    ts = {g: hf.time_graph("single", k, None, img, g, 0, reps=20, samples=5)["mean_us"] for g in (256, 296, 592)}
    k.run(img, 296)
    img.download()
    if x is None:
        x = img.array("bn_x").astype(np.float64).reshape(64, 256, -1)
        mean = x.mean(axis=(0, 2))
        var = x.var(axis=(0, 2))
    ok, err = CK.bn_within_tol(img.array("bn_stats")[:512], mean, var)
    res[(K, T)] = min(ts.values())
    print(json.dumps({"K": K, "threads": T, "regs": k.info.regs, "bps": k.info.blocks_per_sm,
                      "us": {g: round(t, 2) for g, t in ts.items()}, "parity": ok, "rel_err": err}), flush=True)
    del k
del img
best = sorted(res, key=res.get)[:2]
args = types.SimpleNamespace(search_reps=5, granularity=64, waves=[1, 2, 4, 8, 16], split=True, reps=20)
for partner in ("hist", "im2col", "upsample"):
    wb = P.MEMBERS[partner].sizes["full"]()
    img = hf.Image(wa.image).merge(hf.Image(wb.image)).upload()
    sb = P.source("b200", P.MEMBERS[partner].stem)
    for K, T in [(4, 1024)] + [v for v in best if v != (4, 1024)]:
        sa = gen_bn.gen_bn(K, T)
        cfg, _ = bench.search_pair(hf, sa, sb, img, [1024, 768, 512], None, None, args,
                                   natural=256)
        m = bench.build_fused(hf, sa, sb, cfg, img)
        t = hf.time_graph("single", m, None, img, cfg["grid"], 0, reps=20, samples=7)["mean_us"]
        print(json.dumps({"pair": f"bn+{partner}", "K": K, "threads": T, "cfg": cfg, "fused_us": round(t, 2)}),
              flush=True)
        del m
    del img
