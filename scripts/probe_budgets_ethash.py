"""Probe: per-interval register budgets that give the lean Ethash interval MORE registers than its
alone build (64 at 1,024 threads, which spills in the Keccak loop) — the search's budget points
only ever take registers away from a member's alone count. BLAKE2b / BLAKE-256 / SHA-256d + Ethash
at their benched partitions and neighbours, budgets (r1, r2) with r2 in 72..104, against the
uncapped build. Graph protocol. JSON lines (profiles/r02_probe_budgets_ethash.jsonl)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2007_01277_b200 import crypto as CR  # noqa: E402
from paper_2007_01277_b200 import hfuse as hf  # noqa: E402
from paper_2007_01277_b200 import pairs as P  # noqa: E402

COUNTS = {"sha256d": 1 << 24, "blake256": 1 << 24, "blake2b": 1 << 23, "ethash": 1 << 20}
img = hf.Image(CR.workload("ethash", COUNTS["ethash"], 1184, target=1 << 12, npages=33554393).image)
for b in ("sha256d", "blake256", "blake2b"):
    img = img.merge(hf.Image(CR.workload(b, COUNTS[b], 1184, target=1 << 12).image))
img = img.upload()
se = open(os.path.join(P.KERNELS, "b200", "ethash.mk")).read()
POOL = 65536
for a, shapes in (("blake2b", [(256, 640, 148), (256, 512, 148), (384, 512, 148)]),
                  ("blake256", [(256, 768, 148), (128, 768, 148)]),
                  ("sha256d", [(384, 512, 148), (512, 512, 148)])):
    sa = open(os.path.join(P.KERNELS, "b200", a + ".mk")).read()
    for d1, d2, g in shapes:
        m = hf.Module.fused(sa, se, d1, d2, regcap="off", grid=g, specialize=img)
        base = hf.time_graph("single", m, None, img, g, 0, reps=3, samples=5)["mean_us"]
        print(json.dumps({"pair": f"{a}+ethash", "d1": d1, "d2": d2, "grid": g, "budgets": None,
                          "regs": m.info.regs, "us": round(base, 1)}), flush=True)
        del m
        for r2 in (72, 80, 88, 96, 104):
            r1 = (POOL - r2 * d2) // d1 // 8 * 8
            r1 = min(r1, 128)
            if r1 < 32 or d1 % 128 or d2 % 128:
                continue
            try:
                m = hf.Module.fused_regs(sa, se, d1, d2, r1, r2, grid=g, specialize=img)
            except hf.HFuseError as e:
                print(json.dumps({"pair": f"{a}+ethash", "d1": d1, "d2": d2, "budgets": [r1, r2],
                                  "error": str(e)[:160]}), flush=True)
                continue
            t = hf.time_graph("single", m, None, img, g, 0, reps=3, samples=5)["mean_us"]
            print(json.dumps({"pair": f"{a}+ethash", "d1": d1, "d2": d2, "grid": g, "budgets": [r1, r2],
                              "us": round(t, 1), "vs_uncapped": round(base / t, 3)}), flush=True)
            del m
