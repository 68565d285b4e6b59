"""Quick device probe of one DL pair: unfused (sequential / two-stream) vs fused splits.

python scripts/probe_pair.py bn hist [--size full] [--form b200] [--splits 128,256,...]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
from paper_2007_01277_b200 import hfuse as hf  # noqa: E402
from paper_2007_01277_b200.pairs import MEMBERS, source  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("a")
    ap.add_argument("b")
    ap.add_argument("--size", default="full")
    ap.add_argument("--form", default="b200")
    ap.add_argument("--splits", default="128,256,384,512,640,768,896")
    ap.add_argument("--grid", type=int, default=0)
    ap.add_argument("--regcap", default="off")
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    ma, mb = MEMBERS[args.a], MEMBERS[args.b]
    wa, wb = ma.sizes[args.size](0), mb.sizes[args.size](0)
    sa, sb = source(args.form, ma.stem), source(args.form, mb.stem)
    img = hf.Image(wa.image).merge(hf.Image(wb.image)).upload()
    out = {"pair": f"{args.a}+{args.b}", "form": args.form, "size": args.size,
           "bytes": wa.bytes + wb.bytes}
    ka, kb = hf.Module.kernel(sa, grid=args.grid), hf.Module.kernel(sb, grid=args.grid)
    out["regs"] = {"a": ka.info.regs, "b": kb.info.regs}
    for mode in ("sequential", "two_stream"):
        out[mode] = hf.time(mode, ka, kb, img, args.grid, args.grid, reps=args.reps)["median_us"]
    out["a_us"] = hf.time("single", ka, None, img, args.grid, reps=args.reps)["median_us"]
    out["b_us"] = hf.time("single", kb, None, img, args.grid, reps=args.reps)["median_us"]
    out["fused"] = {}
    for d1 in map(int, args.splits.split(",")):
        m = hf.Module.fused(sa, sb, d1, 1024 - d1, regcap=args.regcap, grid=args.grid)
        t = hf.time("single", m, None, img, args.grid, reps=args.reps)["median_us"]
        out["fused"][d1] = {"us": t, "regs": m.info.regs, "bps": m.info.blocks_per_sm}
    best = min(v["us"] for v in out["fused"].values())
    base = min(out["sequential"], out["two_stream"])
    out["best_fused_us"] = best
    out["speedup"] = base / best
    out["hbm_gbs_best"] = out["bytes"] / best / 1e3
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
