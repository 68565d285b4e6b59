"""Probe: the hash members made tunable (their `fixed` 512-thread block dropped) so the partition
search can also size the hash interval, against the fixed form; BLAKE-256 / SHA-256d / BLAKE2b +
Ethash, graph protocol, budgets searched. JSON lines."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2007_01277_b200 import crypto as CR  # noqa: E402
from paper_2007_01277_b200 import hfuse as hf  # noqa: E402
from paper_2007_01277_b200 import pairs as P  # noqa: E402

N = {"sha256d": 1 << 24, "blake2b": 1 << 23, "blake256": 1 << 24, "ethash": 1 << 20}
for a in (sys.argv[1] if len(sys.argv) > 1 else "blake256,sha256d,blake2b").split(","):
    b = "ethash"
    wa = CR.workload(a, N[a], 1184, target=1 << 12)
    wb = CR.workload(b, N[b], 1184, target=1 << 12, npages=33554393)
    img = hf.Image(wa.image).merge(hf.Image(wb.image)).upload()
    sa = open(os.path.join(P.KERNELS, "b200", a + ".mk")).read()
    sb = open(os.path.join(P.KERNELS, "b200", b + ".mk")).read()
    tun = sa.replace(" dims (512, 1, 1) fixed {", " dims (512, 1, 1) {")
    assert tun != sa
    out = {"pair": f"{a}+{b}"}
    for name, src in (("fixed", sa), ("tunable", tun)):
        best = None
        for g in (296, 592):
            for d0 in (768, 896, 1024):
                try:
                    r = hf.search(src, sb, img, d0=d0, grid=g, reps=2, warmup=1, specialize=True, flush_l2=False,
                                  granularity=128, extra_caps=(64, 96, 128), interval_regs=True)
                except hf.HFuseError as e:
                    continue
                if best is None or r["best_time"] < best[0]:
                    best = (r["best_time"], g, d0, r["d1"], r["d2"], r["reg_cap"], r["interval_regs"])
        cfg = {"d1": best[3], "d2": best[4], "reg_cap": best[5], "interval_regs": best[6], "grid": best[1]}
        m = hf.Module.from_config(src, sb, cfg, specialize=img)
        t = hf.time_graph("single", m, None, img, cfg["grid"], 0, reps=3, samples=5)["mean_us"]
        out[name] = {"cfg": cfg, "us": round(t, 1), "screen_ns": best[0]}
        del m
    print(json.dumps(out), flush=True)
    del img
