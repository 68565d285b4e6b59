"""Probe: Ethash with Keccak-f as 24 straight-line rounds (HF_KECCAK_UNROLL=1: immediate round
constants, no round loop) vs the rolled round loop, in the lean (64 registers at 1,024 threads:
ptxas spills 312 B in the rolled loop, 132 B unrolled) and register forms: device parity on a
sub-range, alone at three grids, and fused with BLAKE-256 / SHA-256d / BLAKE2b under the bench's
search. JSON lines (profiles/r02_probe_keccak_unroll.jsonl)."""
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

PAGES = 33554393
COUNTS = {"sha256d": 1 << 24, "blake256": 1 << 24, "blake2b": 1 << 23, "ethash": 1 << 20}


def gen(form, unroll):
    os.environ["HF_KECCAK_UNROLL"] = "1" if unroll else ""
    from paper_2007_01277_b200.kernels import gen_crypto
    g = importlib.reload(gen_crypto)
    return g.gen_ethash() if form == "lean" else g.gen_ethash_reg()


def parity(src, threads, grid=4):
    cnt, n0, tgt = 2600, 99, 1 << 28
    w = CR.workload("ethash", cnt, grid, nonce0=n0, target=tgt, npages=1021)
    img = hf.Image(w.image).upload()
    hf.Module.kernel(src, grid=grid, specialize=img).run(img, grid)
    img.download()
    got = {"cnt": int(img.array("eh_cnt")[0]), "chk": int(img.array("eh_chk")[0]),
           "bmin": [int(x) for x in img.array("eh_bmin")[:grid]]}
    return got == CK.crypto_expected("ethash", cnt, grid, n0, tgt, threads, 1021)


img = hf.Image(CR.workload("ethash", COUNTS["ethash"], 1184, target=1 << 12, npages=PAGES).image)
for b in ("sha256d", "blake256", "blake2b"):
    img = img.merge(hf.Image(CR.workload(b, COUNTS[b], 1184, target=1 << 12).image))
img = img.upload()
srcs = {(f, u): gen(f, u) for f in ("lean", "reg") for u in (False, True)}
for (form, unroll), src in srcs.items():
    k = hf.Module.kernel(src, grid=592, specialize=img)
    thr = 1024 if form == "lean" else 256
    ts = {g: round(hf.time_graph("single", k, None, img, g, 0, reps=3, samples=3)["mean_us"], 1)
          for g in (148, 296, 592)}
    print(json.dumps({"form": form, "unroll": unroll, "parity": parity(src, thr), "regs": k.info.regs,
                      "alone_us": ts}), flush=True)
    del k
only = sys.argv[1].split(",") if len(sys.argv) > 1 else ["blake256", "sha256d", "blake2b"]
for a in only:
    sa = open(os.path.join(P.KERNELS, "b200", a + ".mk")).read()
    for unroll in (False, True):
        sb = srcs[("lean", unroll)]
        traces = []
        for g in (148, 296, 592):
            for d0 in (768, 896, 1024):
                try:
                    r = hf.search(sa, sb, img, d0=d0, grid=g, reps=2, warmup=1, specialize=True, flush_l2=False,
                                  extra_caps=(64, 96, 128), interval_regs=True)
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
        print(json.dumps({"pair": f"{a}+ethash", "unroll": unroll, "cfg": best[0], "fused_us": round(best[1], 1)}),
              flush=True)
