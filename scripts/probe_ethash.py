"""Probe Ethash member variants (v1 per-thread pages vs v2 lane-cooperative) and register caps."""
import json
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
from paper_2007_01277_b200 import crypto as CR  # noqa: E402
from paper_2007_01277_b200 import hfuse as hf  # noqa: E402

G = int(os.environ.get("GRID", "296"))
K = os.path.join(os.path.dirname(__file__), "..", "paper_2007_01277_b200", "kernels", "b200")
v2 = open(os.path.join(K, "ethash.mk")).read()
v1 = open(os.path.join(os.path.dirname(__file__), "ethash_v1.mk")).read()
bl = open(os.path.join(K, "blake256.mk")).read()
we = CR.workload("ethash", 1 << 20, G, npages=1 << 25)
wb = CR.workload("blake256", 1 << 24, G)
img = hf.Image(we.image).merge(hf.Image(wb.image)).upload()
out = {}
for name, src in (("v1", v1), ("v2", v2)):
    for cap in (None, 128, 96, 80, 64):
        try:
            m = hf.Module.kernel(src, regcap=cap, grid=G, specialize=img)
            t = hf.time("single", m, None, img, G, warmup=1, reps=5)["median_us"]
            out[f"{name}_cap{cap}"] = {"us": round(t, 1), "regs": m.info.regs, "bps": m.info.blocks_per_sm,
                                       "mh_s": round((1 << 20) / t, 1)}
        except hf.HFuseError as e:
            out[f"{name}_cap{cap}"] = str(e)[:80]
kb = hf.Module.kernel(bl, grid=G, specialize=img)
out["blake256_us"] = hf.time("single", kb, None, img, G, warmup=1, reps=5)["median_us"]
for name, src in (("v1", v1), ("v2", v2)):
    ke = hf.Module.kernel(src, grid=G, specialize=img)
    out[f"{name}_two_stream"] = hf.time("two_stream", kb, ke, img, G, G, warmup=1, reps=5)["median_us"]
    for cap in (None, 80, 64):
        m = hf.Module.fused(bl, src, 512, 256, regcap=cap or "off", grid=G, specialize=img)
        out[f"{name}_fused_cap{cap}"] = {"us": round(hf.time("single", m, None, img, G, warmup=1, reps=5)["median_us"], 1),
                                         "regs": m.info.regs, "bps": m.info.blocks_per_sm}
print(json.dumps(out, indent=1))
