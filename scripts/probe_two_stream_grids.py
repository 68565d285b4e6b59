"""How much does the two-stream baseline depend on the members' grids? For each DL pair: the
fused kernel at the bench's searched configuration (profiles/r01_bench_full.json), sequential
at each member's best grid alone, and two-stream at every (grid_a, grid_b) combination.
python scripts/probe_two_stream_grids.py > gpurun_out/probe_two_stream_grids.json"""
import json
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
from paper_2007_01277_b200 import hfuse as hf  # noqa: E402
from paper_2007_01277_b200 import pairs as P  # noqa: E402

FLUSH = os.environ.get("HF_PROBE_L2", "steady") == "flush"  # bench default: steady

GRIDS = [296, 592, 1184, 2368]
bench = {r["pair"]: r for r in json.load(open(os.path.join(os.path.dirname(__file__), "..", "profiles",
                                                           "r01_bench_full.json")))["pairs"]}
keys = P.ORDER
img = hf.Image(P.MEMBERS[keys[0]].sizes["full"](0).image)
for k in keys[1:]:
    img.merge(hf.Image(P.MEMBERS[k].sizes["full"](0).image))
img.upload()
src = {k: P.source("b200", P.MEMBERS[k].stem) for k in keys}
mods = {k: hf.Module.kernel(src[k], grid=GRIDS[0], specialize=img) for k in keys}
out = {"alone": {}, "pairs": {}}
best = {}
for k in keys:
    ts = {g: hf.time("single", mods[k], None, img, g, warmup=3, reps=30, flush_l2=FLUSH)["iqm_us"] for g in GRIDS}
    best[k] = min(ts, key=ts.get)
    out["alone"][k] = {str(g): round(t, 2) for g, t in ts.items()}
for a, b in P.PAIRS:
    r = bench[f"{a}+{b}"]
    f = hf.Module.fused(src[a], src[b], r["d1"], r["d2"], regcap=r["reg_cap"] or "off", grid=r["grid"],
                        specialize=img)
    tf = hf.time("single", f, None, img, r["grid"], warmup=5, reps=60, flush_l2=FLUSH)["iqm_us"]
    seq = hf.time("sequential", mods[a], mods[b], img, best[a], best[b], warmup=5, reps=60, flush_l2=FLUSH)["iqm_us"]
    two = {f"{ga}/{gb}": round(hf.time("two_stream", mods[a], mods[b], img, ga, gb, warmup=3, reps=30, flush_l2=FLUSH)["iqm_us"], 2)
           for ga in GRIDS for gb in GRIDS}
    at_best = two[f"{best[a]}/{best[b]}"]
    kbest = min(two, key=two.get)
    row = {"fused": round(tf, 2), "seq": round(seq, 2), "two_at_alone_best": at_best, "two_best": two[kbest],
           "two_best_grids": kbest, "speedup_alone_grids": round(min(seq, at_best) / tf, 3),
           "speedup_best_grids": round(min(seq, two[kbest]) / tf, 3), "two": two}
    out["pairs"][f"{a}+{b}"] = row
    print(f"{a}+{b}", {k: v for k, v in row.items() if k != "two"}, file=sys.stderr, flush=True)
print(json.dumps(out, indent=1))
