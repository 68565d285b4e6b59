"""Launch the benched kernels once each, for ncu (scripts/gpu_ncu_r02.sh): for every DL pair of
profiles/r02_bench_detail.json its two members alone (at the bench's member grids) and the fused
kernel at the bench configuration, on the pair's own tensors, JIT-specialized as bench.py builds
them; then (unless --no-crypto) every crypto pair the same way. Prints the launch order."""
import argparse
import json
import os
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
from paper_2007_01277_b200 import crypto as CR  # noqa: E402
from paper_2007_01277_b200 import hfuse as hf  # noqa: E402
from paper_2007_01277_b200 import pairs as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--detail", default=os.path.join(ROOT, "profiles", "r02_bench_detail.json"))
ap.add_argument("--only", default="", help="comma list of pairs (default all)")
ap.add_argument("--fused-only", action="store_true")
ap.add_argument("--no-crypto", action="store_true")
ap.add_argument("--no-dl", action="store_true")
ap.add_argument("--finalists", action="store_true",
                help="also launch every re-timed finalist configuration of the search (trace 'final' rows)")
args = ap.parse_args()
d = json.load(open(args.detail))
only = set(args.only.split(",")) if args.only else None
order = []


def build(sa, sb, c, img):
    return hf.Module.from_config(sa, sb, c, specialize=img)


for r in d["results"]:
    if args.no_dl or (only and r["pair"] not in only):
        continue
    a, b = r["pair"].split("+")
    img = hf.Image(P.MEMBERS[a].sizes["full"]().image).merge(hf.Image(P.MEMBERS[b].sizes["full"]().image)).upload()
    sa, sb = P.source("b200", P.MEMBERS[a].stem), P.source("b200", P.MEMBERS[b].stem)
    if not args.fused_only:
        for k, s, g in ((a, sa, r["grid_a"]), (b, sb, r["grid_b"])):
            hf.Module.kernel(s, grid=g, specialize=img).run(img, g)
            order.append(f"{r['pair']}:{k}")
    build(sa, sb, r, img).run(img, r["grid"])
    order.append(f"{r['pair']}:fused")
    if args.finalists:
        keys = ("d1", "d2", "reg_cap", "interval_regs", "split_grid", "grid")
        for row in d["search"].get(r["pair"], []):
            if row[0] == "final" and {k: row[1].get(k) for k in keys} != {k: r.get(k) for k in keys}:
                build(sa, sb, row[1], img).run(img, row[1]["grid"])
                order.append(f"{r['pair']}:final:" + json.dumps({k: row[1].get(k) for k in keys}))
    del img
if not args.no_crypto:
    for c in d["crypto"]["pairs"]:
        if c["pair"] == "upsample+blake256" or (only and c["pair"] not in only):
            continue
        a, b = c["pair"].split("+")
        wa = CR.workload(a, c["per_rank_nonces"][a], max(c["grid"], c["grid_a"], c["grid_b"]), target=1 << 12)
        wb = CR.workload(b, c["per_rank_nonces"][b], max(c["grid"], c["grid_a"], c["grid_b"]), target=1 << 12,
                         npages=33554393)
        img = hf.Image(wa.image).merge(hf.Image(wb.image)).upload()
        fa, fb = c.get("forms") or (a, b)  # the member forms the bench fused
        sa = open(os.path.join(P.KERNELS, "b200", fa + ".mk")).read()
        sb = open(os.path.join(P.KERNELS, "b200", fb + ".mk")).read()
        if not args.fused_only:  # each member in the form its unfused baseline ran (bench baseline_forms)
            forms = c.get("baseline_forms") or {}
            for k, g in ((a, c["grid_a"]), (b, c["grid_b"])):
                s = open(os.path.join(P.KERNELS, "b200", forms.get(k, k) + ".mk")).read()
                hf.Module.kernel(s, grid=g, specialize=img).run(img, g)
                order.append(f"{c['pair']}:{k}")
        build(sa, sb, c, img).run(img, c["grid"])
        order.append(f"{c['pair']}:fused")
        del img
import ctypes  # noqa: E402
ctypes.CDLL("libcudart.so.12").cudaDeviceSynchronize()
print(json.dumps(order))
