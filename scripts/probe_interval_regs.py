"""Probe per-interval register budgets (setmaxnreg) on the crypto pairs and C4: for each
partition, sweep (regs1, regs2) over the largest pool one CTA per SM allows and time the
fused kernel against the same pair fused with one whole-kernel cap and run unfused."""
import json
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
from paper_2007_01277_b200 import crypto as CR  # noqa: E402
from paper_2007_01277_b200 import hfuse as hf  # noqa: E402
from paper_2007_01277_b200 import pairs as P  # noqa: E402

G = int(os.environ.get("GRID", "296"))
K = os.path.join(P.KERNELS, "b200")
src = {k: open(os.path.join(K, k + ".mk")).read() for k in CR.MEMBERS}
src["upsample"] = P.source("b200", "upsample")
COUNTS = {"sha256d": 1 << 24, "blake2b": 1 << 23, "blake256": 1 << 24, "ethash": 1 << 20}


def budgets(d1, d2, lo=24):
    launch = (65536 // (d1 + d2)) // 8 * 8
    pool = launch * (d1 + d2)
    out = []
    for r1 in range(lo, 257, 8):
        r2 = min(256, (pool - r1 * d1) // d2 // 8 * 8)
        if r2 >= 24:
            out.append((r1, r2))
    return out


def t(m, img):
    return round(hf.time("single", m, None, img, G, warmup=2, reps=7)["iqm_us"], 1)


res = {}
pairs = os.environ.get("PAIRS", "blake256+ethash,sha256d+blake2b,upsample+blake256").split(",")
for pair in pairs:
    a, b = pair.split("+")
    ws = []
    for k in (a, b):
        if k == "upsample":
            ws.append(P.MEMBERS["upsample"].sizes["full"](0).image)
        else:
            ws.append(CR.workload(k, COUNTS[k] if pair != "upsample+blake256" else 1 << 21, G,
                                  npages=1 << 25).image)
    img = hf.Image(ws[0]).merge(hf.Image(ws[1])).upload()
    ka = hf.Module.kernel(src[a], grid=G, specialize=img)
    kb = hf.Module.kernel(src[b], grid=G, specialize=img)
    r = {"a_regs": ka.info.regs, "b_regs": kb.info.regs,
         "seq": round(hf.time("sequential", ka, kb, img, G, G, warmup=2, reps=7)["iqm_us"], 1),
         "two": round(hf.time("two_stream", ka, kb, img, G, G, warmup=2, reps=7)["iqm_us"], 1), "rows": []}
    splits = {"blake256+ethash": [(512, 128), (512, 256), (512, 384), (512, 512)],
              "sha256d+blake2b": [(512, 512)],
              "upsample+blake256": [(256, 512), (384, 512), (512, 512)]}[pair]
    for d1, d2 in splits:
        for cap in ("off", 64, 96):
            try:
                m = hf.Module.fused(src[a], src[b], d1, d2, regcap=cap, grid=G, specialize=img)
                r["rows"].append({"d1": d1, "d2": d2, "cap": cap, "regs": m.info.regs, "us": t(m, img)})
            except hf.HFuseError as e:
                r["rows"].append({"d1": d1, "d2": d2, "cap": cap, "err": str(e)[:100]})
        bs = budgets(d1, d2)
        step = max(1, len(bs) // 6)
        for r1, r2 in bs[::step]:
            try:
                m = hf.Module.fused_regs(src[a], src[b], d1, d2, r1, r2, grid=G, specialize=img)
                i = m.info
                r["rows"].append({"d1": d1, "d2": d2, "r1": r1, "r2": r2, "launch": i.launch_regs,
                                  "local": i.local_bytes, "bps": i.blocks_per_sm, "us": t(m, img)})
            except hf.HFuseError as e:
                r["rows"].append({"d1": d1, "d2": d2, "r1": r1, "r2": r2, "err": str(e)[:100]})
        print(pair, d1, d2, json.dumps(r["rows"][-8:]), flush=True)
    res[pair] = r
    del img
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/probe_interval_regs.json", "w"), indent=1)
print(json.dumps({p: {k: v for k, v in r.items() if k != "rows"} for p, r in res.items()}))
