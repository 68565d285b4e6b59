"""Cache-operator probe: the five DL members alone and the ten fused pairs (at the bench's
searched configurations, profiles/r01_bench_full.json) with the vector moves' cache operator set
by HF_VLOAD_HINT / HF_VSTORE_HINT (read once per process by the emitter), against the unfused
sequential / two-stream launch under the same hints. One JSON line per process.
HF_VLOAD_HINT=cs python scripts/probe_hints.py >> gpurun_out/probe_hints.jsonl"""
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
out = {"load": os.environ.get("HF_VLOAD_HINT", ""), "store": os.environ.get("HF_VSTORE_HINT", ""),
       "alone": {}, "pairs": {}}
alone = {}
for k in keys:
    m = hf.Module.kernel(src[k], grid=GRIDS[0], specialize=img)
    ts = {g: hf.time("single", m, None, img, g, warmup=3, reps=20, flush_l2=FLUSH)["iqm_us"] for g in GRIDS}
    g = min(ts, key=ts.get)
    alone[k] = (m, g)
    out["alone"][k] = round(ts[g], 2)
for a, b in P.PAIRS:
    r = bench[f"{a}+{b}"]
    f = hf.Module.fused(src[a], src[b], r["d1"], r["d2"], regcap=r["reg_cap"] or "off", grid=r["grid"],
                        specialize=img)
    tf = hf.time("single", f, None, img, r["grid"], warmup=3, reps=40, flush_l2=FLUSH)["iqm_us"]
    (ma, ga), (mb, gb) = alone[a], alone[b]
    seq = hf.time("sequential", ma, mb, img, ga, gb, warmup=3, reps=40, flush_l2=FLUSH)["iqm_us"]
    two = hf.time("two_stream", ma, mb, img, ga, gb, warmup=3, reps=40, flush_l2=FLUSH)["iqm_us"]
    out["pairs"][f"{a}+{b}"] = {"fused": round(tf, 2), "seq": round(seq, 2), "two": round(two, 2),
                                "speedup": round(min(seq, two) / tf, 3)}
img.download()
out["digest"] = img.digest_hex()
print(json.dumps(out), flush=True)
