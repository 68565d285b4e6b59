"""Probe: the lean-register Ethash form (HF_ETHASH_FORM=lean: cp.async DAG ring + Keccak seed
parked in shared memory, ~64-80 registers) against the register form (127 registers), alone and
fused with BLAKE-256 under the bench's search (per-interval budgets). Device parity of every
form on a sub-range against crypto_ref first. Graph protocol. JSON lines on stdout."""
import importlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import check as CK  # noqa: E402
from paper_2007_01277_b200 import crypto as CR  # noqa: E402
from paper_2007_01277_b200 import hfuse as hf  # noqa: E402
from paper_2007_01277_b200 import pairs as P  # noqa: E402

NP = 33554393


def gen(form, tmax):
    os.environ["HF_ETHASH_FORM"], os.environ["HF_ETHASH_TMAX"] = form, str(tmax)
    from paper_2007_01277_b200.kernels import gen_crypto
    return importlib.reload(gen_crypto).gen_ethash()


def parity(src, threads, grid):
    cnt, n0, tgt = 384, 777, 1 << 28
    w = CR.workload("ethash", cnt, grid, nonce0=n0, target=tgt, npages=1021)
    img = hf.Image(w.image).upload()
    hf.Module.kernel(src, grid=grid, specialize=img).run(img, grid)
    img.download()
    got = {"cnt": int(img.array("eh_cnt")[0]), "chk": int(img.array("eh_chk")[0]),
           "bmin": [int(x) for x in img.array("eh_bmin")[:grid]]}
    return got == CK.crypto_expected("ethash", cnt, grid, n0, tgt, threads, 1021)


N = 1 << 20
wb = CR.workload("ethash", N, 1184, target=1 << 12, npages=NP)
COUNTS = {"blake256": 1 << 24, "sha256d": 1 << 24, "blake2b": 1 << 23}
partners = (sys.argv[2].split(",") if len(sys.argv) > 2 else ["blake256"])
img = hf.Image(wb.image)
for a in partners:
    img = img.merge(hf.Image(CR.workload(a, COUNTS[a], 1184, target=1 << 12).image))
img = img.upload()
forms = [("reg", 512, 256), ("lean", 768, 768), ("lean", 1024, 1024), ("lean", 896, 896)]
only = sys.argv[1:] and set(sys.argv[1].split(","))
for (form, tmax, block), a in [(f, a) for a in partners for f in forms]:
    tag = f"{form}{tmax}"
    if only and tag not in only:
        continue
    blake = open(os.path.join(P.KERNELS, "b200", a + ".mk")).read()
    src = gen(form, tmax)
    if a == partners[0]:
        print(json.dumps({"form": tag, "parity": parity(src, block, 3)}), flush=True)
    k = hf.Module.kernel(src, grid=592, specialize=img)
    for g in ((148, 296, 592) if a == partners[0] else ()):
        t = hf.time_graph("single", k, None, img, g, 0, reps=3, samples=3)["mean_us"]
        print(json.dumps({"form": tag, "grid": g, "block": block, "regs": k.info.regs, "bps": k.info.blocks_per_sm,
                          "us": round(t, 1), "dag_gbs": round(N * 8192 / (t * 1e3), 1)}), flush=True)
    traces = []
    for g in (148, 296):
        for d0 in (768, 896, 1024):
            if form == "lean" and d0 - 128 > tmax:
                continue
            try:
                r = hf.search(blake, src, img, d0=d0, grid=g, reps=2, warmup=1, specialize=True, flush_l2=False,
                              extra_caps=(64, 96, 128), interval_regs=True)
            except hf.HFuseError as e:
                print(json.dumps({"form": tag, "d0": d0, "grid": g, "err": str(e)[:160]}), flush=True)
                continue
            traces += [(g, x["d1"], x["d2"], x["reg_cap"], x["us"]) for x in r["trace"] if x["d2"] <= tmax or form == "reg"]
    best = []
    for g, d1, d2, cap, us in sorted(traces, key=lambda t: t[4])[:4]:
        cfg = {"d1": d1, "d2": d2, "grid": g, "reg_cap": None, "interval_regs": None}
        if "/" in str(cap):
            cfg["interval_regs"] = [int(x) for x in str(cap).split("/")]
        elif cap not in ("none", None):
            cfg["reg_cap"] = int(cap)
        try:
            m = hf.Module.from_config(blake, src, cfg, specialize=img)
        except hf.HFuseError as e:
            print(json.dumps({"form": tag, "cfg": cfg, "err": str(e)[:160]}), flush=True)
            continue
        t = hf.time_graph("single", m, None, img, g, 0, reps=3, samples=5)["mean_us"]
        print(json.dumps({"form": tag, "partner": a, "fused": cfg, "screen_us": round(us, 1), "us": round(t, 1),
                          "regs": m.info.regs}), flush=True)
        del m
