"""Probe: SHA-256d with its rotates on the ALU pipe (funnel shifts, the round-1 member) vs on the
FMA pipe (HF_SHA_PIPES=fma: x * 2^k and mulhi_u(x, 2^k) with the power in a register; ptxas emits
one IMAD.WIDE.U32 per rotate half-pair), alone and fused with each partner hash under the bench's
crypto search (interval budgets). Device parity of each form on a sub-range first. Graph protocol.
JSON lines (profiles/r02_probe_sha_pipes.jsonl)."""
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


def gen(pipes):
    os.environ["HF_SHA_PIPES"] = pipes
    from paper_2007_01277_b200.kernels import gen_crypto
    return importlib.reload(gen_crypto).gen_sha256d()


def parity(src, grid=3):
    cnt, n0, tgt = 4096, 777, 1 << 28
    w = CR.workload("sha256d", cnt, grid, nonce0=n0, target=tgt)
    img = hf.Image(w.image).upload()
    hf.Module.kernel(src, grid=grid, specialize=img).run(img, grid)
    img.download()
    got = {"cnt": int(img.array("sh_cnt")[0]), "chk": int(img.array("sh_chk")[0]),
           "bmin": [int(x) for x in img.array("sh_bmin")[:grid]]}
    return got == CK.crypto_expected("sha256d", cnt, grid, n0, tgt, 512, 1 << 10)


partners = sys.argv[1].split(",") if len(sys.argv) > 1 else ["blake256", "blake2b", "ethash"]
img = hf.Image(CR.workload("sha256d", COUNTS["sha256d"], 1184, target=1 << 12).image)
for b in partners:
    img = img.merge(hf.Image(CR.workload(b, COUNTS[b], 1184, target=1 << 12, npages=33554393).image))
img = img.upload()
srcs = {"alu": gen("alu"), "fma": gen("fma")}
for form, src in srcs.items():
    k = hf.Module.kernel(src, grid=592, specialize=img)
    ts = {g: round(hf.time_graph("single", k, None, img, g, 0, reps=3, samples=3)["mean_us"], 1) for g in (296, 592, 1184)}
    print(json.dumps({"form": form, "parity": parity(src), "regs": k.info.regs, "bps": k.info.blocks_per_sm,
                      "alone_us": ts}), flush=True)
    del k
for b in partners:
    sb = open(os.path.join(P.KERNELS, "b200", b + ".mk")).read()
    for form, src in srcs.items():
        traces = []
        for g in ((148, 296, 592) if b == "ethash" else (296, 592)):
            for d0 in ((768, 896, 1024) if b == "ethash" else (1024,)):
                try:
                    r = hf.search(src, sb, img, d0=d0, grid=g, reps=2, warmup=1, specialize=True, flush_l2=False,
                                  extra_caps=(64, 96, 128) if b == "ethash" else (), interval_regs=True)
                except hf.HFuseError:
                    continue
                traces += [(g, x["d1"], x["d2"], x["reg_cap"], x["us"]) for x in r["trace"]]
        best = None
        for g, d1, d2, cap, us in sorted(traces, key=lambda t: t[4])[:3]:
            cfg = {"d1": d1, "d2": d2, "grid": g, "reg_cap": None, "interval_regs": None}
            if "/" in str(cap):
                cfg["interval_regs"] = [int(x) for x in str(cap).split("/")]
            elif cap not in ("none", None):
                cfg["reg_cap"] = int(cap)
            try:
                m = hf.Module.from_config(src, sb, cfg, specialize=img)
            except hf.HFuseError:
                continue
            t = hf.time_graph("single", m, None, img, g, 0, reps=3, samples=5)["mean_us"]
            if best is None or t < best[1]:
                best = (cfg, t)
            del m
        print(json.dumps({"form": form, "pair": f"sha256d+{b}", "cfg": best[0], "fused_us": round(best[1], 1)}),
              flush=True)
