"""BatchNorm forms for fusion: block-per-channel (batchnorm.mk) vs warp-balanced
(batchnorm_warp.mk), alone and fused (device search) with each DL partner, against the
sequential / two-stream unfused pair at each variant's best grid."""
import json
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
from paper_2007_01277_b200 import hfuse as hf  # noqa: E402
from paper_2007_01277_b200 import pairs as P  # noqa: E402

GRIDS = [296, 592, 1184, 2368]
keys = ["bn", "hist", "im2col", "maxpool", "upsample"]
# the warp-level hand-off needs (grid / C + 2) * 32 partial slots per channel
img = hf.Image(P._bn(64, 256, 56 * 56, slots=512)(0).image)
for k in keys[1:]:
    img.merge(hf.Image(P.MEMBERS[k].sizes["full"](0).image))
img.upload()
forms = {"block": P.source("b200", "batchnorm"), "warp": P.source("b200", "batchnorm_warp")}
# timing-only diagnostic (not a correct BN): no hand-off at all, partial stores only
DIAG = {"warp_nohandoff": forms["warp"].replace("atomic_add_release(bn_cnt[c], 1);", "")
        .replace("load_relaxed(bn_cnt[c]) == parts", "parts == -7")}
src = {k: P.source("b200", P.MEMBERS[k].stem) for k in keys[1:]}


def best_alone(s):
    m = hf.Module.kernel(s, grid=GRIDS[0], specialize=img)
    ts = {g: hf.time("single", m, None, img, g, warmup=2, reps=10)["iqm_us"] for g in GRIDS}
    g = min(ts, key=ts.get)
    return m, g, ts


out = {}
alone = {}
for name, s in list(forms.items()) + list(DIAG.items()) + list(src.items()):
    m, g, ts = best_alone(s)
    alone[name] = (m, g)
    out[f"alone_{name}"] = {str(k): round(v, 2) for k, v in ts.items()}
    print(name, out[f"alone_{name}"], flush=True)
# the warp form's result must equal the block form's within tolerance (different order)
import numpy as np  # noqa: E402
res = {}
for name in forms:
    m, g = alone[name]
    m.run(img, g)
    img.download()
    res[name] = np.array(img.array("bn_stats"))
out["max_rel_diff"] = float(np.max(np.abs(res["warp"] - res["block"]) / np.maximum(1, np.abs(res["block"]))))
print("max_rel_diff", out["max_rel_diff"], flush=True)
for partner in keys[1:]:
    for name, s in forms.items():
        best = None
        for g in GRIDS:
            r = hf.search(s, src[partner], img, d0=1024, grid=g, reps=5, warmup=2, specialize=True, granularity=64)
            if best is None or r["best_time"] < best[0]["best_time"]:
                best = (r, g)
        r, g = best
        ma, ga = alone[name]
        mb, gb = alone[partner]
        seq = hf.time("sequential", ma, mb, img, ga, gb, warmup=2, reps=20)["iqm_us"]
        two = hf.time("two_stream", ma, mb, img, ga, gb, warmup=2, reps=20)["iqm_us"]
        f = hf.Module.fused(s, src[partner], r["d1"], r["d2"], regcap=r["reg_cap"] or "off", grid=g, specialize=img)
        tf = hf.time("single", f, None, img, g, warmup=2, reps=20)["iqm_us"]
        out[f"{name}+{partner}"] = {"grid": g, "d1": r["d1"], "cap": r["reg_cap"], "fused": round(tf, 2),
                                    "seq": round(seq, 2), "two": round(two, 2),
                                    "speedup": round(min(seq, two) / tf, 3)}
        print(name, partner, out[f"{name}+{partner}"], flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe_bn_warp.json", "w"), indent=1)
