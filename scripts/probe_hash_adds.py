"""Probe: the ALU-pipe-bound hash members with their adds moved onto the FMA pipe (MK+ fma_add =
IMAD a, one, b): SHA-256d (HF_SHA_ADDS=fma: every round/schedule add) and BLAKE-256
(HF_B256_ADDS: "a" = the a = a + b + (m ^ c) adds, "c" = the c = c + d adds). Each form: device
parity on a sub-range, time alone at three grids; then each crypto pair fused with the base and
the FMA-add forms under the bench's search (interval budgets), top-3 re-timed. Graph protocol.
JSON lines (profiles/r02_probe_hash_adds.jsonl)."""
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

COUNTS = {"sha256d": 1 << 24, "blake256": 1 << 24, "blake2b": 1 << 23, "ethash": 1 << 20}
PFX = {"sha256d": "sh", "blake256": "bl"}
FORMS = {"sha256d": {"base": {}, "fma": {"HF_SHA_ADDS": "fma"}},
         "blake256": {"base": {}, "a": {"HF_B256_ADDS": "a"}, "ac": {"HF_B256_ADDS": "ac"}}}


def gen(kind, env):
    for k in ("HF_SHA_ADDS", "HF_B256_ADDS"):
        os.environ.pop(k, None)
    os.environ.update(env)
    from paper_2007_01277_b200.kernels import gen_crypto
    g = importlib.reload(gen_crypto)
    return {"sha256d": g.gen_sha256d, "blake256": g.gen_blake256}[kind]()


def parity(kind, src, grid=3):
    cnt, n0, tgt = 4096, 777, 1 << 28
    w = CR.workload(kind, cnt, grid, nonce0=n0, target=tgt)
    img = hf.Image(w.image).upload()
    hf.Module.kernel(src, grid=grid, specialize=img).run(img, grid)
    img.download()
    p = PFX[kind]
    got = {"cnt": int(img.array(f"{p}_cnt")[0]), "chk": int(img.array(f"{p}_chk")[0]),
           "bmin": [int(x) for x in img.array(f"{p}_bmin")[:grid]]}
    return got == CK.crypto_expected(kind, cnt, grid, n0, tgt, 512, 1 << 10)


img = hf.Image(CR.workload("sha256d", COUNTS["sha256d"], 1184, target=1 << 12).image)
for b in ("blake256", "blake2b", "ethash"):
    img = img.merge(hf.Image(CR.workload(b, COUNTS[b], 1184, target=1 << 12, npages=33554393).image))
img = img.upload()
srcs = {kind: {f: gen(kind, env) for f, env in forms.items()} for kind, forms in FORMS.items()}
for kind, forms in srcs.items():
    for form, src in forms.items():
        k = hf.Module.kernel(src, grid=592, specialize=img)
        ts = {g: round(hf.time_graph("single", k, None, img, g, 0, reps=3, samples=3)["mean_us"], 1)
              for g in (296, 592, 1184)}
        print(json.dumps({"member": kind, "form": form, "parity": parity(kind, src), "regs": k.info.regs,
                          "bps": k.info.blocks_per_sm, "alone_us": ts}), flush=True)
        del k


def src_of(kind, form):
    if kind in srcs:
        return srcs[kind][form]
    return open(os.path.join(P.KERNELS, "b200", kind + ".mk")).read()


PAIRS = [("sha256d", "blake256"), ("blake256", "ethash"), ("sha256d", "ethash"), ("blake256", "blake2b"),
         ("sha256d", "blake2b")]
only = sys.argv[1].split(",") if len(sys.argv) > 1 else None
for a, b in PAIRS:
    if only and f"{a}+{b}" not in only:
        continue
    combos = [("base", "base")]
    fa = [f for f in FORMS.get(a, {}) if f != "base"] or ["base"]
    fb = [f for f in FORMS.get(b, {}) if f != "base"] or ["base"]
    combos += [(x, y) for x in fa[:1] for y in fb[:1]]
    for x, y in combos:
        sa, sb = src_of(a, x), src_of(b, y)
        traces = []
        for g in ((148, 296, 592) if b == "ethash" else (296, 592)):
            for d0 in ((768, 896, 1024) if b == "ethash" else (1024,)):
                try:
                    r = hf.search(sa, sb, img, d0=d0, grid=g, reps=2, warmup=1, specialize=True, flush_l2=False,
                                  extra_caps=(64, 96, 128) if b == "ethash" else (), interval_regs=True)
                except hf.HFuseError:
                    continue
                traces += [(g, t["d1"], t["d2"], t["reg_cap"], t["us"]) for t in r["trace"]]
        best = None
        for g, d1, d2, cap, us in sorted(traces, key=lambda t: t[4])[:3]:
            cfg = {"d1": d1, "d2": d2, "grid": g, "reg_cap": None, "interval_regs": None}
            if "/" in str(cap):
                cfg["interval_regs"] = [int(v) for v in str(cap).split("/")]
            elif cap not in ("none", None):
                cfg["reg_cap"] = int(cap)
            try:
                m = hf.Module.from_config(sa, sb, cfg, specialize=img)
            except hf.HFuseError:
                continue
            t = hf.time_graph("single", m, None, img, g, 0, reps=3, samples=5)["mean_us"]
            if best is None or t < best[1]:
                best = (cfg, t)
            del m
        print(json.dumps({"pair": f"{a}+{b}", "forms": [x, y], "cfg": best[0], "fused_us": round(best[1], 1)}),
              flush=True)
