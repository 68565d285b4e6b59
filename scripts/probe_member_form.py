"""Compare two B200 forms of one DL member: alone (best grid) and fused (device search over
grids) with each other DL member, against the unfused sequential / two-stream pair.
python scripts/probe_member_form.py MEMBER ALT.mk [ALT2.mk ...] [out.json]"""
import json
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
from paper_2007_01277_b200 import hfuse as hf  # noqa: E402
from paper_2007_01277_b200 import pairs as P  # noqa: E402

FLUSH = os.environ.get("HF_PROBE_L2", "steady") == "flush"  # bench default: steady

member = sys.argv[1]
alts = [a for a in sys.argv[2:] if a.endswith(".mk")]
outs = [a for a in sys.argv[2:] if a.endswith(".json")]
out_path = outs[0] if outs else f"gpurun_out/probe_{member}_form.json"
GRIDS = [296, 592, 1184, 2368]
keys = P.ORDER
img = hf.Image(P.MEMBERS[keys[0]].sizes["full"](0).image)
for k in keys[1:]:
    img.merge(hf.Image(P.MEMBERS[k].sizes["full"](0).image))
img.upload()
src = {k: P.source("b200", P.MEMBERS[k].stem) for k in keys}
forms = {"current": src[member]}
for a in alts:
    forms["alt" if len(alts) == 1 else os.path.basename(a)[:-3]] = open(a).read()
out = {"alone": {}, "pairs": {}}
alone = {}
for name, s in list(forms.items()) + [(k, src[k]) for k in keys if k != member]:
    m = hf.Module.kernel(s, grid=GRIDS[0], specialize=img)
    ts = {g: hf.time("single", m, None, img, g, warmup=2, reps=10, flush_l2=FLUSH)["iqm_us"] for g in GRIDS}
    g = min(ts, key=ts.get)
    alone[name] = (m, g)
    out["alone"][name] = {"regs": m.info.regs, **{str(k): round(v, 2) for k, v in ts.items()}}
    print(name, out["alone"][name], flush=True)
# same outputs (bit-exact forms): digest of the image after each form
digs = {}
for name in forms:
    m, g = alone[name]
    m.run(img, g)
    img.download()
    digs[name] = img.digest_hex()
out["same_digest"] = len(set(digs.values())) == 1
print("same digest", out["same_digest"], flush=True)
for partner in [k for k in keys if k != member]:
    for name, s in forms.items():
        a_src, b_src = (s, src[partner]) if keys.index(member) < keys.index(partner) else (src[partner], s)
        best = None
        for g in GRIDS:
            r = hf.search(a_src, b_src, img, d0=1024, grid=g, reps=5, warmup=2, specialize=True, granularity=64, flush_l2=FLUSH)
            if best is None or r["best_time"] < best[0]["best_time"]:
                best = (r, g)
        r, g = best
        (ma, ga), (mb, gb) = alone[name], alone[partner]
        seq = hf.time("sequential", ma, mb, img, ga, gb, warmup=2, reps=20, flush_l2=FLUSH)["iqm_us"]
        two = hf.time("two_stream", ma, mb, img, ga, gb, warmup=2, reps=20, flush_l2=FLUSH)["iqm_us"]
        f = hf.Module.fused(a_src, b_src, r["d1"], r["d2"], regcap=r["reg_cap"] or "off", grid=g, specialize=img)
        tf = hf.time("single", f, None, img, g, warmup=2, reps=20, flush_l2=FLUSH)["iqm_us"]
        out["pairs"][f"{name}+{partner}"] = {"grid": g, "d1": r["d1"], "cap": r["reg_cap"], "fused": round(tf, 2),
                                             "seq": round(seq, 2), "two": round(two, 2),
                                             "speedup": round(min(seq, two) / tf, 3)}
        print(name, partner, out["pairs"][f"{name}+{partner}"], flush=True)
os.makedirs(os.path.dirname(out_path) or ".", exist_ok=True)
json.dump(out, open(out_path, "w"), indent=1)
