"""Does the order of the ten kernels in the PDL step matter? The fused kernels at the bench's
configurations (profiles/r01_bench_full.json) and the twenty unfused kernels at their best grids,
timed as programmatic dependent launches on one stream in several orders (K = 30 steps each).
python scripts/probe_step_order.py > gpurun_out/probe_step_order.json"""
import json
import os
import random
import sys

import torch

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
from paper_2007_01277_b200 import hfuse as hf  # noqa: E402
from paper_2007_01277_b200 import pairs as P  # noqa: E402

bench = json.loads(open(os.path.join(os.path.dirname(__file__), "..", "profiles", "r01_bench_full.json"))
                   .read().strip().splitlines()[-1])
img = hf.Image(P.MEMBERS["bn"].sizes["full"](0).image)
for k in P.ORDER[1:]:
    img.merge(hf.Image(P.MEMBERS[k].sizes["full"](0).image))
img.upload()
stream = torch.cuda.current_stream()
src = {k: P.source("b200", P.MEMBERS[k].stem) for k in P.ORDER}
mgrid = {k: int(min(v, key=v.get)) for k, v in bench["config"]["member_grid_us"].items()}
unf = {k: hf.Module.kernel(src[k], grid=mgrid[k], specialize=img) for k in P.ORDER}
fused = {}
for p in bench["pairs"]:
    a, b = p["pair"].split("+")
    fused[p["pair"]] = (hf.Module.fused(src[a], src[b], p["d1"], p["d2"], regcap=p["reg_cap"] or "off",
                                        grid=p["grid"], specialize=img), p["grid"])
wfrac = {p["pair"]: 0 for p in bench["pairs"]}
for p in bench["pairs"]:
    a, b = p["pair"].split("+")
    w = P.MEMBERS[a].sizes["full"](0).write + P.MEMBERS[b].sizes["full"](0).write
    wfrac[p["pair"]] = w / p["bytes"]
base = [p["pair"] for p in bench["pairs"]]
by_w = sorted(base, key=wfrac.get)
inter = [x for pair in zip(by_w[:5], reversed(by_w[5:])) for x in pair]
orders = {"bench": base, "reversed": base[::-1], "write_ascending": by_w, "read_write_interleaved": inter}
rng = random.Random(7)
for i in range(3):
    o = base[:]
    rng.shuffle(o)
    orders[f"random{i}"] = o


def timed(fn, steps=30, warm=5):
    for _ in range(warm):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(stream)
    for _ in range(steps):
        fn()
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / steps


out = {"orders": orders, "fused_us": {}, "unfused_us": {}}
for rep in range(2):
    for name, o in orders.items():
        def fstep(o=o):
            for pr in o:
                m, g = fused[pr]
                m.run(img, g, stream, overlap=True)

        def ustep(o=o):
            for pr in o:
                a, b = pr.split("+")
                unf[a].run(img, mgrid[a], stream, overlap=True)
                unf[b].run(img, mgrid[b], stream, overlap=True)
        out["fused_us"].setdefault(name, []).append(round(timed(fstep), 1))
        out["unfused_us"].setdefault(name, []).append(round(timed(ustep), 1))
for name in orders:
    print(name, out["fused_us"][name], out["unfused_us"][name], file=sys.stderr, flush=True)
print(json.dumps(out, indent=1))
